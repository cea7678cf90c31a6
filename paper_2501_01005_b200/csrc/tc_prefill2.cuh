// tc_prefill2.cuh — ragged paged prefill on tcgen05 with two softmax warpgroups (T_q = 64/128).
//
// Same math and plan contract as tc_prefill.cuh (one work item = (request, kv head, q tile of
// 128 head-fused rows, kv chunk) from Algorithm 1, App. A head fusion, online softmax P:95,
// writethrough App. D.2), re-organised so the tensor core never waits for one softmax:
//   * the CTA's plan queue is split into two item streams (even / odd queue positions), one per
//     softmax warpgroup (WG); each WG owns its S/P and O accumulators in TMEM (4 x 128 columns);
//   * a dedicated MMA warp walks the two streams' KV tiles in a fixed interleaved order and
//     issues S_w = Q_w K^T as soon as K has landed and WG w released its S buffer, and
//     O_w += P_w V with P_w read straight from TMEM (TS-MMA; P overwrites the consumed S columns);
//   * producers: warp 0 loads Q (per WG) and K, warp 1 loads V, through separate rings, in the
//     same interleaved order; per page one TMA box {64 d, B_c tokens} per 64-column half, page
//     coordinate from the BSR indices (§3.2.1);
//   * softmax reads S from TMEM twice (max pass, exp pass) to keep registers low, uses ex2.approx
//     with the scale folded into an FFMA, lazy O rescale (threshold 2^8, exact).
// Ordering facts used: tcgen05 MMAs of one thread complete in issue order, so S_w(t+1) ready
// implies PV_w(t) done (O_w quiescent while WG w runs its softmax).
#pragma once
#include "tc_decode.cuh"
#include "tc_kernels.hpp"

namespace bsra {

namespace pre2 {
constexpr int kTile = 128;
constexpr int kKStages = 3;
constexpr int kVStages = 2;
constexpr int kHalf = 128 * 128;   // 16 KB: 128 rows x 128 B
constexpr int kOp = 2 * kHalf;     // 32 KB operand (128 x 128 bf16, two SW128 halves)
constexpr int kOffQ = 0;           // [2 WGs]
constexpr int kOffK = 2 * kOp;
constexpr int kOffV = kOffK + kKStages * kOp;
constexpr int kOffBar = kOffV + kVStages * kOp;
constexpr int kSmemBytes = kOffBar + 512 + 1024;
constexpr int kThreads = 384;      // warps 0 Q+K producer, 1 V producer, 2 MMA, 3 idle, 4-7 WG0, 8-11 WG1
constexpr uint32_t kTmemCols = 512;  // S/P_w at w*128, O_w at 256 + w*128
constexpr float kRescaleThresh = 8.f;
}  // namespace pre2

// Walks one WG's item stream (queue positions it0+w, it0+w+2, ...) tile by tile.
struct ItemStream {
  int it, it1;
  int ti;
  DecItem d;
  __device__ __forceinline__ void init(const PlanView& pv, int g, int first, int end) {
    it = first;
    it1 = end;
    ti = 0;
    skip_empty(pv, g);
  }
  __device__ __forceinline__ void skip_empty(const PlanView& pv, int g) {
    while (it < it1) {
      d = dec_item(pv, it, g);
      if (d.ntiles > 0) return;
      it += 2;
    }
  }
  __device__ __forceinline__ bool alive() const { return it < it1; }
  // advance one tile; returns true if an item boundary was crossed
  __device__ __forceinline__ bool advance(const PlanView& pv, int g) {
    if (++ti < d.ntiles) return false;
    ti = 0;
    it += 2;
    skip_empty(pv, g);
    return true;
  }
};

// Deterministic interleave of the two streams: alternate while both are alive.
struct Interleave {
  ItemStream s[2];
  int turn = 0;
  __device__ __forceinline__ void init(const PlanView& pv, int g, int it0, int it1) {
    s[0].init(pv, g, it0, it1);
    s[1].init(pv, g, it0 + 1, it1);
    turn = 0;
  }
  __device__ __forceinline__ int pick() const {  // -1 when both exhausted
    if (s[0].alive() && s[1].alive()) return turn;
    if (s[0].alive()) return 0;
    if (s[1].alive()) return 1;
    return -1;
  }
  __device__ __forceinline__ void step(const PlanView& pv, int g, int w) {
    const bool both = s[0].alive() && s[1].alive();
    s[w].advance(pv, g);
    if (both) turn ^= 1;
  }
};

template <int kMask>
__global__ void __launch_bounds__(pre2::kThreads, 1) tc_prefill2_kernel(const __grid_constant__ TcParams tp) {
  using namespace pre2;
  const AttnParams& p = tp.p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* full_k = bar;                    // [kKStages]
  uint64_t* empty_k = full_k + kKStages;     // [kKStages]
  uint64_t* full_v = empty_k + kKStages;     // [kVStages]
  uint64_t* empty_v = full_v + kVStages;     // [kVStages]
  uint64_t* full_q = empty_v + kVStages;     // [2] per WG
  uint64_t* empty_q = full_q + 2;            // [2]
  uint64_t* bar_s = empty_q + 2;             // [2] S_w ready
  uint64_t* p_ready = bar_s + 2;             // [2] P_w written (128 arrivals)
  uint64_t* bar_o = p_ready + 2;             // [2] last PV of WG w's item done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_o + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PlanView pv = load_plan(p.plan);
  const int g = p.g;
  const int it0 = pv.cta_indptr[blockIdx.x], it1 = pv.cta_indptr[blockIdx.x + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKStages; ++s) {
      ptx::mbar_init(&full_k[s], 1);
      ptx::mbar_init(&empty_k[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      ptx::mbar_init(&full_v[s], 1);
      ptx::mbar_init(&empty_v[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      ptx::mbar_init(&full_q[w], 1);
      ptx::mbar_init(&empty_q[w], 1);
      ptx::mbar_init(&bar_s[w], 1);
      ptx::mbar_init(&p_ready[w], 128);
      ptx::mbar_init(&bar_o[w], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int B = tp.box_tok;

  if (warp == 0 || warp == 1) {
    // ===================== producers: warp 0 = Q + K, warp 1 = V =====================
    const bool isK = warp == 0;
    if (lane == 0) {
      if (isK) {
        ptx::tma_prefetch_desc(&tp.tq);
        ptx::tma_prefetch_desc(&tp.tk);
      } else {
        ptx::tma_prefetch_desc(&tp.tv);
      }
    }
    Interleave il;
    il.init(pv, g, it0, it1);
    int stage = 0;
    uint32_t ephase = 1;
    uint32_t qphase[2] = {1, 1};
    const int nst = isK ? kKStages : kVStages;
    uint64_t* fullx = isK ? full_k : full_v;
    uint64_t* emptyx = isK ? empty_k : empty_v;
    const CUtensorMap* tm = isK ? &tp.tk : &tp.tv;
    const int ring = isK ? kOffK : kOffV;
    for (int w = il.pick(); w >= 0; w = il.pick()) {
      const DecItem& d = il.s[w].d;
      const int ti = il.s[w].ti;
      if (isK && ti == 0 && lane == 0) {  // Q of WG w's next item
        ptx::mbar_wait(&empty_q[w], qphase[w]);
        qphase[w] ^= 1;
        ptx::mbar_arrive_expect_tx(&full_q[w], kOp);
        const int head0 = d.kvh * g + (g > 128 ? d.row0 % g : 0);
        const int tok0 = (int)d.qo_begin + d.row0 / g;
        uint8_t* qdst = smem + kOffQ + w * kOp;
        ptx::tma_load_3d(qdst, &tp.tq, &full_q[w], 0, head0, tok0);
        ptx::tma_load_3d(qdst + kHalf, &tp.tq, &full_q[w], 64, head0, tok0);
      }
      const int64_t t0 = d.kb + (int64_t)ti * kTile;
      const int n = (int)imin64(kTile, d.ke - t0);
      const int nsub = (n + B - 1) / B;
      int page = 0, off = 0;
      if (lane < nsub) {
        const int64_t tok = t0 + (int64_t)lane * B;
        page = __ldg(p.page_indices + d.page_begin + tok / p.page_size);
        off = (int)(tok % p.page_size);
      }
      if (lane == 0) {
        ptx::mbar_wait(&emptyx[stage], ephase);
        ptx::mbar_arrive_expect_tx(&fullx[stage], (uint32_t)nsub * B * 256);
      }
      __syncwarp();
      if (lane < nsub) {
        uint8_t* dst = smem + ring + stage * kOp + lane * B * 128;
        ptx::tma_load_4d(dst, tm, &fullx[stage], 0, d.kvh, off, page);
        ptx::tma_load_4d(dst + kHalf, tm, &fullx[stage], 64, d.kvh, off, page);
      }
      __syncwarp();
      if (++stage == nst) {
        stage = 0;
        ephase ^= 1;
      }
      il.step(pv, g, w);
    }
  } else if (warp == 2) {
    // ===================== MMA issuer (one elected lane) =====================
    const uint32_t fmt = tp.f16 ? 0u : 1u;
    const uint32_t idS = ptx::idesc_f16(fmt, 128, kTile, 0, 0);  // A = Q (K-major), B = K (K-major)
    const uint32_t idO = ptx::idesc_f16(fmt, 128, 128, 0, 1);    // A = P (TMEM), B = V (MN-major)
    const uint32_t sbase = ptx::smem_u32(smem);
    // Two cursors over the same interleaved tile sequence: `sq` issues S (K ring order), `il`
    // issues PV (V ring order). A WG has one S buffer, so S of its next tile waits until the PV
    // of its current tile has been issued (in-order tensor pipe => no WAR hazard on TMEM).
    Interleave il, sq;
    il.init(pv, g, it0, it1);
    sq.init(pv, g, it0, it1);
    int kst = 0, vst = 0;
    uint32_t kph = 0, vph = 0;
    uint32_t qph[2] = {0, 0}, pph[2] = {0, 0};
    bool q_loaded[2] = {false, false};
    int pending[2] = {0, 0};  // WG w has an S issued whose PV is not yet issued
    auto issue_S = [&](int w) {
      const DecItem& d = sq.s[w].d;
      const bool last = sq.s[w].ti + 1 == d.ntiles;
      if (!q_loaded[w]) {  // first tile of a new item: wait for its Q
        if (lane == 0) ptx::mbar_wait(&full_q[w], qph[w]);
        qph[w] ^= 1;
        q_loaded[w] = true;
      }
      if (lane == 0) {
        ptx::mbar_wait(&full_k[kst], kph);
        ptx::tc_fence_after();
        const uint32_t qa = sbase + kOffQ + w * kOp, ka = sbase + kOffK + kst * kOp;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = ptx::smem_desc_sw128(qa + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
          const uint64_t b = ptx::smem_desc_sw128(ka + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
          ptx::mma_f16_ss(tmem + w * 128, a, b, idS, kk > 0);
        }
        ptx::mma_commit(&empty_k[kst]);
        ptx::mma_commit(&bar_s[w]);
        if (last) ptx::mma_commit(&empty_q[w]);  // last S of the item: Q buffer free
      }
      __syncwarp();
      if (last) q_loaded[w] = false;
      if (++kst == kKStages) {
        kst = 0;
        kph ^= 1;
      }
      pending[w] = 1;
      sq.step(pv, g, w);
    };
    for (int w = il.pick(); w >= 0; w = il.pick()) {
      for (int sw = sq.pick(); sw >= 0 && !pending[sw]; sw = sq.pick()) issue_S(sw);
      const DecItem d = il.s[w].d;
      const int ti = il.s[w].ti;
      const int64_t t0 = d.kb + (int64_t)ti * kTile;
      const int n = (int)imin64(kTile, d.ke - t0);
      // wait V, zero rows past the chunk (0 * garbage could be NaN)
      ptx::mbar_wait(&full_v[vst], vph);
      if (n < kTile) {
        uint8_t* vS = smem + kOffV + vst * kOp;
        for (int rr = n + lane; rr < kTile; rr += 32) {
          uint4* v0 = reinterpret_cast<uint4*>(vS + rr * 128);
          uint4* v1 = reinterpret_cast<uint4*>(vS + kHalf + rr * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v0[j] = make_uint4(0, 0, 0, 0);
            v1[j] = make_uint4(0, 0, 0, 0);
          }
        }
        ptx::fence_proxy_async();
        __syncwarp();
      }
      ptx::mbar_wait(&p_ready[w], pph[w]);
      pph[w] ^= 1;
      if (lane == 0) {
        ptx::tc_fence_after();
        const uint32_t va = sbase + kOffV + vst * kOp;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t b = ptx::smem_desc_sw128(va + kk * 2048, kHalf, 1024);
          ptx::mma_f16_ts(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, b, idO, (ti > 0 || kk > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&empty_v[vst]);
        if (ti + 1 == d.ntiles) ptx::mma_commit(&bar_o[w]);
      }
      __syncwarp();
      if (++vst == kVStages) {
        vst = 0;
        vph ^= 1;
      }
      pending[w] = 0;
      il.step(pv, g, w);
    }
  } else if (warp >= 4) {
    // ===================== softmax warpgroups =====================
    const int w = (warp - 4) >> 2;        // WG index
    const int q4 = warp & 3;              // TMEM lane quarter
    const int r = q4 * 32 + lane;         // fused row of the tile
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_addr + w * 128;
    const uint32_t tO = tmem + lane_addr + 256 + w * 128;
    const float sc = p.scale_log2;
    uint32_t sph = 0, oph = 0;
    for (int it = it0 + w; it < it1; it += 2) {
      const DecItem d = dec_item(pv, it, g);
      const bool row_ok = r < d.nrows;
      const int f = d.row0 + r;
      const int tok = f / g, head = d.kvh * g + f % g;
      const int64_t lim = kMask == 1 ? d.lk - d.lq + tok : d.ke - 1;
      const int64_t mbase = kMask == 2 ? p.mask_indptr[d.req] + (int64_t)tok * d.lk : 0;
      float m = -INFINITY, l = 0.f;
      for (int ti = 0; ti < d.ntiles; ++ti) {
        const int64_t t0 = d.kb + (int64_t)ti * kTile;
        const int n = (int)imin64(kTile, d.ke - t0);
        const int64_t vis_end = row_ok ? (kMask == 1 ? imin64(lim + 1, t0 + n) : t0 + n) : t0;
        const int nvis = (int)(vis_end > t0 ? vis_end - t0 : 0);
        const bool need_mask = kMask == 2 || nvis < kTile;
        ptx::mbar_wait(&bar_s[w], sph);
        sph ^= 1;
        ptx::tc_fence_after();
        // ---- pass 1: raw row max
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float s[32];
          ptx::tmem_ld32(tS + c * 32, s);
          ptx::tmem_ld_wait();
          if (need_mask) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              bool vis = c * 32 + j < nvis;
              if (kMask == 2) vis = vis && mask_bit(p.mask, mbase + t0 + c * 32 + j);
              s[j] = vis ? s[j] : -INFINITY;
            }
          }
          float a0 = fmaxf(s[0], s[1]), a1 = fmaxf(s[2], s[3]), a2 = fmaxf(s[4], s[5]), a3 = fmaxf(s[6], s[7]);
#pragma unroll
          for (int j = 8; j < 32; j += 4) {
            a0 = fmaxf(a0, s[j]);
            a1 = fmaxf(a1, s[j + 1]);
            a2 = fmaxf(a2, s[j + 2]);
            a3 = fmaxf(a3, s[j + 3]);
          }
          mx = fmaxf(mx, fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
        }
        const float mt = mx * sc;
        float alpha = 1.f;
        bool rescale = false;
        if (mt > m + kRescaleThresh) {
          if (m != -INFINITY) {
            alpha = ptx_ex2(m - mt);
            rescale = true;
          }
          m = mt;
        }
        // O_w is quiescent here (PV_w(t-1) completed before S_w(t) did)
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float ov[32];
            ptx::tmem_ld32(tO + c * 32, ov);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] *= alpha;
            uint32_t* ou = reinterpret_cast<uint32_t*>(ov);
            ptx::tmem_st16(tO + c * 32, ou);
            ptx::tmem_st16(tO + c * 32 + 16, ou + 16);
          }
        }
        // ---- pass 2: P = 2^(s*scale - m) packed to 16-bit pairs, written over the consumed S columns
        const float mneg = m == -INFINITY ? 0.f : -m;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float s[32];
          ptx::tmem_ld32(tS + c * 32, s);
          ptx::tmem_ld_wait();
          if (need_mask) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              bool vis = c * 32 + j < nvis;
              if (kMask == 2) vis = vis && mask_bit(p.mask, mbase + t0 + c * 32 + j);
              s[j] = vis ? s[j] : -INFINITY;
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float p0 = ptx_ex2(fmaf(s[j], sc, mneg));
            const float p1 = ptx_ex2(fmaf(s[j + 1], sc, mneg));
            rs0 += p0;
            rs1 += p1;
            if (tp.f16) {
              __half2 h = __floats2half2_rn(p0, p1);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          ptx::tmem_st16(tS + c * 16, pk);
        }
        l = l * alpha + (rs0 + rs1);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_ready[w]);
      }
      // ---- epilogue: wait for the item's last PV, normalise, write
      if (d.ntiles > 0) {
        ptx::mbar_wait(&bar_o[w], oph);
        oph ^= 1;
        ptx::tc_fence_after();
      }
      const bool empty_row = !(l > 0.f);
      const float inv = empty_row ? 0.f : 1.f / l;
      const float lse = empty_row ? -INFINITY : (m + __log2f(l)) * kLn2;
      const int64_t orow = (d.qo_begin + tok) * p.H_qo + head;
      const int64_t prow = (int64_t)d.slot * p.T_slot + r;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        float ov[32];
        if (d.ntiles > 0) {
          ptx::tmem_ld32(tO + c0, ov);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) ov[j] = 0.f;
        }
        if (!row_ok) continue;
        if (d.slot >= 0 || p.o_f32) {
          float* dstf = d.slot >= 0 ? p.part_o + prow * 128 + c0 : reinterpret_cast<float*>(p.o) + orow * 128 + c0;
          float4* dst = reinterpret_cast<float4*>(dstf);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(ov[4 * j] * inv, ov[4 * j + 1] * inv, ov[4 * j + 2] * inv, ov[4 * j + 3] * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.o) + orow * 128 + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t wv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a0 = ov[8 * j + 2 * e] * inv, a1 = ov[8 * j + 2 * e + 1] * inv;
              if (tp.f16) {
                __half2 h = __floats2half2_rn(a0, a1);
                wv[e] = *reinterpret_cast<uint32_t*>(&h);
              } else {
                __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
                wv[e] = *reinterpret_cast<uint32_t*>(&h);
              }
            }
            dst[j] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
      if (row_ok) {
        if (d.slot >= 0) p.part_lse[prow] = lse;
        else if (p.lse) p.lse[orow] = lse;
      }
      ptx::tc_fence_before();  // O_w reads done before this WG's next p_ready (next item's PV)
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc<kTmemCols>(tmem);
}

template <int kMask>
inline cudaError_t launch_prefill2_t(const TcParams& tp, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_prefill2_kernel<kMask>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pre2::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  tc_prefill2_kernel<kMask><<<grid, pre2::kThreads, pre2::kSmemBytes, st>>>(tp);
  return cudaGetLastError();
}

}  // namespace bsra
