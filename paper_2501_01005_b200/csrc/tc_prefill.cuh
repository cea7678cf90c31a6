// tc_prefill.cuh — ragged paged prefill attention on tcgen05 tensor cores (T_q = 64 / 128).
//
// One work item = (request, kv head, q tile of 128 head-fused rows, kv chunk) from Algorithm 1.
// Head-group fusion (App. A): fused row f <-> token f / g, qo head kvh*g + f % g, so
// the 128 rows of a tile are 128/g tokens x g heads and every K/V tile loaded serves all of them.
//     S[128 rows x 128 tok] = Q[128 x D] . K^T          (tcgen05, fp32 in TMEM, double-buffered)
//     O[128 x D]           += P[128 x 128] . V          (P bf16/fp16 in smem, O accumulates in TMEM)
// Warp roles (one CTA per SM, persistent over the plan queue):
//   warps 0, 5 TMA producers: Q tile per item (double-buffered) + K pages, and V pages, through
//              separate 2-deep rings (K is freed as soon as its S MMA completes); per page one box
//              {64 d, B_c tokens} per 64-column half of the 4-D pool view, the page coordinate
//              taken from the BSR indices (§3.2.1).
//   warps 1-4  128 threads, thread = fused row = TMEM lane: the row max / sum are thread-local
//              (no shuffles), online softmax in the log2 domain with lazy O rescaling
//              (threshold 2^8; exact because o and lse use the same max). Causal / custom masks
//              are applied per element only on tiles that cross a row's limit.
// Epilogue: unsplit rows write o / lse (App. D.2), split rows fp32 partial slots.
#pragma once
#include <cstdlib>

#include "tc_decode.cuh"
#include "tc_kernels.hpp"
#include "tc_prefill2.cuh"

namespace bsra {

namespace pre {
constexpr int kM = 128;                       // fused rows per tile (MMA M)
constexpr int kTile = 128;                    // kv tokens per tile (MMA N of S, K of PV)
constexpr int kStages = 2;                    // depth of the K ring and of the V ring
constexpr int kHalf = 128 * 128;              // 128 rows x 64 cols x 2 B = 16 KB
constexpr int kOp = 2 * kHalf;                // one 128 x 128 operand: 32 KB
constexpr int kOffQ = 0;                      // 2 Q buffers
constexpr int kOffK = 2 * kOp;                // K ring
constexpr int kOffV = kOffK + kStages * kOp;  // V ring
constexpr int kOffP = kOffV + kStages * kOp;  // P (A operand of PV)
constexpr int kOffBar = kOffP + kOp;
constexpr int kSmemBytes = kOffBar + 256 + 1024;
constexpr int kThreads = 192;                 // warp 0: Q+K producer, warps 1-4: softmax/MMA, warp 5: V producer
constexpr uint32_t kTmemCols = 512;           // S buffers at 0 / 128, O at 256
constexpr float kRescaleThresh = 8.f;
}  // namespace pre

// One producer warp's share of a KV tile: lane j loads sub-block j (one page, or 128 tokens of
// a page >= 128) — both 64-column halves — with the page coordinate from the BSR indices.
// (page, in-page offset) of this lane's sub-block; loaded before the producer waits for a free
// stage so the index latency overlaps the wait.
__device__ __forceinline__ void kv_tile_coords(const AttnParams& p, const DecItem& d, int64_t t0, int n, int B,
                                               int lane, int& page, int& off) {
  const int nsub = (n + B - 1) / B;
  page = 0;
  off = 0;
  if (lane < nsub) {
    const int64_t tok = t0 + (int64_t)lane * B;
    if (p.kv_ragged) {  // contiguous KV: token coordinate, no page table
      off = (int)(d.page_begin + tok);
    } else {
      page = __ldg(p.page_indices + d.page_begin + tok / p.page_size);
      off = (int)(tok % p.page_size);
    }
  }
}
__device__ __forceinline__ void load_kv_tile(const CUtensorMap* tm, uint8_t* dst, uint64_t* bar, const DecItem& d,
                                             int n, int B, int lane, int half_bytes, int page, int off) {
  const int nsub = (n + B - 1) / B;
  if (lane < nsub) {
    uint8_t* kd = dst + lane * B * 128;
    ptx::tma_load_4d(kd, tm, bar, 0, d.kvh, off, page);
    ptx::tma_load_4d(kd + half_bytes, tm, bar, 64, d.kvh, off, page);
  }
}

template <int kMask>
__global__ void __launch_bounds__(pre::kThreads, 1) tc_prefill_kernel(const __grid_constant__ TcParams tp) {
  using namespace pre;
  const AttnParams& p = tp.p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* full_k = bar;                  // [kStages]
  uint64_t* empty_k = bar + kStages;       // [kStages]  freed by the S MMA
  uint64_t* full_v = bar + 2 * kStages;    // [kStages]
  uint64_t* empty_v = bar + 3 * kStages;   // [kStages]  freed by the PV MMA
  uint64_t* full_q = bar + 4 * kStages;    // [2]
  uint64_t* empty_q = full_q + 2;          // [2]
  uint64_t* bar_s = empty_q + 2;           // [2]
  uint64_t* bar_pv = bar_s + 2;            // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_pv + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PlanView pv = load_plan(p.plan);
  const int g = p.g;
  const int it0 = pv.cta_indptr[blockIdx.x], it1 = pv.cta_indptr[blockIdx.x + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full_k[s], 1);
      ptx::mbar_init(&empty_k[s], 1);
      ptx::mbar_init(&full_v[s], 1);
      ptx::mbar_init(&empty_v[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&full_q[b], 1);
      ptx::mbar_init(&empty_q[b], 1);
      ptx::mbar_init(&bar_s[b], 1);
    }
    ptx::mbar_init(bar_pv, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 5) {
    // ===================== TMA producers (warp 0: Q + K, warp 5: V) =====================
    const bool isK = warp == 0;
    if (lane == 0) {
      if (isK) {
        ptx::tma_prefetch_desc(&tp.tq);
        ptx::tma_prefetch_desc(&tp.tk);
      } else {
        ptx::tma_prefetch_desc(&tp.tv);
      }
    }
    const int B = tp.box_tok;
    int stage = 0;
    uint32_t ephase = 1;
    uint32_t qphase[2] = {1, 1};
    int qb = 0;
    uint64_t* fullx = isK ? full_k : full_v;
    uint64_t* emptyx = isK ? empty_k : empty_v;
    const CUtensorMap* tm = isK ? &tp.tk : &tp.tv;
    const int ring = isK ? kOffK : kOffV;
    for (int it = it0; it < it1; ++it) {
      const DecItem d = dec_item(pv, it, g);
      if (isK) {
        if (lane == 0) {
          ptx::mbar_wait(&empty_q[qb], qphase[qb]);
          ptx::mbar_arrive_expect_tx(&full_q[qb], kOp);
          const int head0 = d.kvh * g + (g > kM ? d.row0 % g : 0);
          const int tok0 = (int)d.qo_begin + d.row0 / g;
          uint8_t* qdst = smem + kOffQ + qb * kOp;
          ptx::tma_load_3d(qdst, &tp.tq, &full_q[qb], 0, head0, tok0);
          ptx::tma_load_3d(qdst + kHalf, &tp.tq, &full_q[qb], 64, head0, tok0);
        }
        qphase[qb] ^= 1;
        qb ^= 1;
      }
      for (int ti = 0; ti < d.ntiles; ++ti) {
        const int64_t t0 = d.kb + (int64_t)ti * kTile;
        const int n = (int)imin64(kTile, d.ke - t0);
        const int nsub = (n + B - 1) / B;
        int page, off;
        kv_tile_coords(p, d, t0, n, B, lane, page, off);
        if (lane == 0) {
          ptx::mbar_wait(&emptyx[stage], ephase);
          ptx::mbar_arrive_expect_tx(&fullx[stage], (uint32_t)nsub * B * 256);
        }
        __syncwarp();
        load_kv_tile(tm, smem + ring + stage * kOp, &fullx[stage], d, n, B, lane, kHalf, page, off);
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          ephase ^= 1;
        }
      }
    }
  } else {
    // ===================== softmax / MMA / epilogue warps =====================
    const int ct = threadIdx.x - 32;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // fused row within the tile = TMEM lane
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    const uint32_t tO = tmem + lane_addr + 256;
    const uint32_t fmt = tp.f16 ? 0u : 1u;
    const uint32_t idS = ptx::idesc_f16(fmt, kM, kTile, 0, 0);  // A = Q (K-major), B = K (K-major)
    const uint32_t idO = ptx::idesc_f16(fmt, kM, 128, 0, 1);    // A = P (K-major), B = V (MN-major)
    const uint32_t sbase = ptx::smem_u32(smem);
    int stage = 0;
    uint32_t fphase = 0;
    uint32_t sph[2] = {0, 0}, pvph = 0;
    bool pv_pending = false;
    int sbuf = 0;
    uint32_t qphase[2] = {0, 0};
    int qb = 0;

    // elected thread: S(b) = Q K(st)^T; frees the K stage and signals the S buffer on completion
    auto issue_S = [&](int st, int b, uint32_t qaddr) {
      ptx::tc_fence_after();
      const uint32_t ka = sbase + kOffK + st * kOp;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t a = ptx::smem_desc_sw128(qaddr + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = ptx::smem_desc_sw128(ka + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
        ptx::mma_f16_ss(tmem + b * 128, a, bd, idS, kk > 0);
      }
      ptx::mma_commit(&empty_k[st]);
      ptx::mma_commit(&bar_s[b]);
    };
    auto wait_pv = [&]() {
      if (pv_pending) {
        ptx::mbar_wait(bar_pv, pvph);
        pvph ^= 1;
        pv_pending = false;
      }
    };

    for (int it = it0; it < it1; ++it) {
      const DecItem d = dec_item(pv, it, g);
      const uint32_t qaddr = sbase + kOffQ + qb * kOp;
      const bool row_ok = r < d.nrows;
      const int f = d.row0 + r;
      const int tok = f / g, head = d.kvh * g + f % g;
      // visible iff t <= lim (causal) / mask bit (custom); rows past the tile are never visible
      const int64_t lim = kMask == 1 ? d.lk - d.lq + tok : d.ke - 1;
      const int64_t mbase = kMask == 2 ? p.mask_indptr[d.req] + (int64_t)tok * d.lk : 0;
      float m = -INFINITY, l = 0.f;
      ptx::mbar_wait(&full_q[qb], qphase[qb]);
      qphase[qb] ^= 1;
      bool next_issued = false;
      if (d.ntiles > 0 && ct == 0) {
        ptx::mbar_wait(&full_k[stage], fphase);
        issue_S(stage, sbuf, qaddr);
      }
      for (int ti = 0; ti < d.ntiles; ++ti) {
        const int64_t t0 = d.kb + (int64_t)ti * kTile;
        const int n = (int)imin64(kTile, d.ke - t0);
        const int nstage = stage + 1 == kStages ? 0 : stage + 1;
        const uint32_t nfphase = nstage == 0 ? fphase ^ 1 : fphase;
        next_issued = false;
        if (ct == 0 && ti + 1 < d.ntiles && ptx::mbar_test_wait(&full_k[nstage], nfphase)) {
          issue_S(nstage, sbuf ^ 1, qaddr);
          next_issued = true;
        }
        ptx::mbar_wait(&bar_s[sbuf], sph[sbuf]);
        sph[sbuf] ^= 1;
        ptx::tc_fence_after();
        float s[kTile];
        const uint32_t tS = tmem + lane_addr + sbuf * 128;
        ptx::tmem_ld32(tS + 0, s);
        ptx::tmem_ld32(tS + 32, s + 32);
        ptx::tmem_ld32(tS + 64, s + 64);
        ptx::tmem_ld32(tS + 96, s + 96);
        ptx::tmem_ld_wait();
        // ---- mask (only where the tile crosses this row's limit), raw row max
        const int64_t vis_end = row_ok ? (kMask == 1 ? imin64(lim + 1, t0 + n) : t0 + n) : t0;  // exclusive
        const int nvis = (int)(vis_end > t0 ? vis_end - t0 : 0);
        if (kMask == 2 || nvis < kTile) {
#pragma unroll
          for (int j = 0; j < kTile; ++j) {
            bool vis = j < nvis;
            if (kMask == 2) vis = vis && mask_bit(p.mask, mbase + t0 + j);
            s[j] = vis ? s[j] : -INFINITY;
          }
        }
        float mx8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mx8[k] = s[k];
#pragma unroll
        for (int j = 8; j < kTile; ++j) mx8[j & 7] = fmaxf(mx8[j & 7], s[j]);
        const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                 fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float mt = mraw * p.scale_log2;  // scale > 0: max commutes with scaling; -inf stays -inf
        float alpha = 1.f;
        bool rescale = false;
        if (mt > m + kRescaleThresh) {
          if (m != -INFINITY) {
            alpha = ptx_ex2(m - mt);
            rescale = true;
          }
          m = mt;
        }
        const float mneg = m == -INFINITY ? 0.f : -m;  // p = 2^(s*scale - m); masked s = -inf -> 0
        const float sc = p.scale_log2;
        float rs4[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pw[kTile / 2];  // P packed as bf16x2 / f16x2 (halves the live registers)
#pragma unroll
        for (int j = 0; j < kTile; j += 2) {
          const float p0 = ptx_ex2(fmaf(s[j], sc, mneg));
          const float p1 = ptx_ex2(fmaf(s[j + 1], sc, mneg));
          rs4[(j >> 1) & 3] += p0 + p1;
          if (tp.f16) {
            __half2 h = __floats2half2_rn(p0, p1);
            pw[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
          } else {
            __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
            pw[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
          }
        }
        l = l * alpha + ((rs4[0] + rs4[1]) + (rs4[2] + rs4[3]));
        if (n < kTile && r >= n) {  // V rows past the chunk -> 0 (0 * garbage would poison O)
          ptx::mbar_wait(&full_v[stage], fphase);
          uint8_t* vS = smem + kOffV + stage * kOp;
          uint4 z = make_uint4(0, 0, 0, 0);
          uint4* v0 = reinterpret_cast<uint4*>(vS + r * 128);
          uint4* v1 = reinterpret_cast<uint4*>(vS + kHalf + r * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v0[j] = z;
            v1[j] = z;
          }
        }
        wait_pv();  // PV(i-1) has finished reading P, and O is quiescent
        // tcgen05.ld/st are warp-collective: the whole warp rescales if any of its rows must
        if (__any_sync(0xffffffffu, rescale)) {
          ptx::tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < 128; c0 += 32) {
            float ov[32];
            ptx::tmem_ld32(tO + c0, ov);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] *= alpha;
            uint32_t* ou = reinterpret_cast<uint32_t*>(ov);
            ptx::tmem_st16(tO + c0, ou);
            ptx::tmem_st16(tO + c0 + 16, ou + 16);
          }
          ptx::tmem_st_wait();
        }
        // ---- P (bf16/fp16) -> smem, K-major SW128 A operand
        {
          uint8_t* prow = smem + kOffP + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
          for (int c = 0; c < 16; ++c) {  // 16 chunks of 8 tokens
            const int a = c >> 3, cc = c & 7;
            *reinterpret_cast<uint4*>(prow + a * kHalf + ((cc ^ (r & 7)) << 4)) =
                make_uint4(pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
          }
        }
        ptx::fence_proxy_async();
        ptx::tc_fence_before();
        ptx::named_bar_sync(1, 128);
        if (ct == 0) {
          ptx::tc_fence_after();
          ptx::mbar_wait(&full_v[stage], fphase);
          const uint32_t pa = sbase + kOffP;
          const uint32_t va = sbase + kOffV + stage * kOp;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t a = ptx::smem_desc_sw128(pa + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
            const uint64_t b = ptx::smem_desc_sw128(va + kk * 2048, kHalf, 1024);
            ptx::mma_f16_ss(tmem + 256, a, b, idO, (ti > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty_v[stage]);
          ptx::mma_commit(bar_pv);
          if (!next_issued && ti + 1 < d.ntiles) {
            ptx::mbar_wait(&full_k[nstage], nfphase);
            issue_S(nstage, sbuf ^ 1, qaddr);
          }
        }
        pv_pending = true;
        sbuf ^= 1;
        stage = nstage;
        fphase = nfphase;
      }
      wait_pv();
      if (ct == 0) ptx::mbar_arrive(&empty_q[qb]);
      qb ^= 1;
      // ---- epilogue: thread r owns its whole row (TMEM loads warp-uniform, stores per row)
      {
        const bool empty_row = !(l > 0.f);
        const float inv = empty_row ? 0.f : p.v_scale / l;  // v_scale: fp8 KV (R28), else 1
        const float lse = empty_row ? -INFINITY : (m + __log2f(l)) * kLn2;
        if (d.ntiles > 0) ptx::tc_fence_after();
        if (d.slot < 0) {
          const int64_t orow = (d.qo_begin + tok) * p.H_qo + head;
#pragma unroll
          for (int c0 = 0; c0 < 128; c0 += 32) {
            float ov[32];
            if (d.ntiles > 0) {
              ptx::tmem_ld32(tO + c0, ov);
              ptx::tmem_ld_wait();
            }
            if (!row_ok) continue;
            if (p.o_f32) {
              float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.o) + orow * 128 + c0);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(ov[4 * j] * inv, ov[4 * j + 1] * inv, ov[4 * j + 2] * inv, ov[4 * j + 3] * inv);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.o) + orow * 128 + c0);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float a0 = ov[8 * j + 2 * e] * inv, a1 = ov[8 * j + 2 * e + 1] * inv;
                  if (tp.f16) {
                    __half2 h = __floats2half2_rn(a0, a1);
                    w[e] = *reinterpret_cast<uint32_t*>(&h);
                  } else {
                    __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
                    w[e] = *reinterpret_cast<uint32_t*>(&h);
                  }
                }
                dst[j] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          }
          if (p.lse && row_ok) p.lse[orow] = lse;
        } else {
          const int64_t prow = (int64_t)d.slot * p.T_slot + r;
#pragma unroll
          for (int c0 = 0; c0 < 128; c0 += 32) {
            float ov[32];
            if (d.ntiles > 0) {
              ptx::tmem_ld32(tO + c0, ov);
              ptx::tmem_ld_wait();
            }
            if (!row_ok) continue;
            float4* dst = reinterpret_cast<float4*>(p.part_o + prow * 128 + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(ov[4 * j] * inv, ov[4 * j + 1] * inv, ov[4 * j + 2] * inv, ov[4 * j + 3] * inv);
          }
          if (row_ok) p.part_lse[prow] = lse;
        }
      }
      if (d.slot >= 0 && p.fused_merge) {  // split item: fused contraction (see merge.cuh)
        volatile int* s_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
        if (tp.f16) fused_contraction<__half, 128>(p, pv, d.slot, r, 128, 1, s_flag);
        else fused_contraction<__nv_bfloat16, 128>(p, pv, d.slot, r, 128, 1, s_flag);
      }
      ptx::tc_fence_before();
      ptx::named_bar_sync(1, 128);  // TMEM reads of O done before the next item's first PV
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<kTmemCols>(tmem);
}

template <int kMask>
inline cudaError_t launch_prefill_t(const TcParams& tp, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(tc_prefill_kernel<kMask>, cudaFuncAttributeMaxDynamicSharedMemorySize, pre::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  tc_prefill_kernel<kMask><<<grid, pre::kThreads, pre::kSmemBytes, st>>>(tp);
  return cudaGetLastError();
}

bool make_q_map_ext(CUtensorMap* m, const void* q, bool f16, int H_qo, int64_t N, int hb, int tb);
bool make_kv_maps(TcParams& tp, const AttnParams& p, const TcLaunch& L, int B);

inline int tc_prefill_launch(const AttnParams& p, const TcLaunch& L, cudaStream_t st, const char** name,
                             const char** why, int B) {
  const int g = p.g;
  if (g > 128) {
    *why = "group size > 128";
    return 0;
  }
  TcParams tp;
  memset(&tp, 0, sizeof(tp));
  tp.p = p;
  tp.box_tok = B;
  tp.q_hb = g;
  tp.q_tb = 128 / g;
  tp.f16 = L.f16;
  tp.pdl = L.pdl;
  static const int dbg = getenv("BSRA_DEBUG_PREFILL") ? atoi(getenv("BSRA_DEBUG_PREFILL")) : 0;
  tp.dbg = dbg;  // timing experiments only (never set in tests / bench)
  if (!make_q_map_ext(&tp.tq, p.q, L.f16, p.H_qo, L.total_qo, tp.q_hb, tp.q_tb) || !make_kv_maps(tp, p, L, B)) {
    *why = "cuTensorMapEncodeTiled failed";
    return -1;
  }
  cudaError_t e;
  static const bool v1 = getenv("BSRA_PREFILL_V1") != nullptr;  // A/B against the one-warpgroup kernel
  const bool variants = p.window > 0 || p.soft_cap > 0.f || p.alibi;  // the v1 A/B kernel has no variant support
  if (L.T_q == 256) {  // paired: both softmax WGs on one item, every K/V tile feeds 256 rows
    switch (L.mask) {
      case 0: e = launch_prefill2_t<0, true>(tp, L.grid, st); break;
      case 1: e = launch_prefill2_t<1, true>(tp, L.grid, st); break;
      default: e = launch_prefill2_t<2, true>(tp, L.grid, st); break;
    }
  } else if (v1 && !variants) {
    switch (L.mask) {
      case 0: e = launch_prefill_t<0>(tp, L.grid, st); break;
      case 1: e = launch_prefill_t<1>(tp, L.grid, st); break;
      default: e = launch_prefill_t<2>(tp, L.grid, st); break;
    }
  } else {
    switch (L.mask) {
      case 0: e = launch_prefill2_t<0, false>(tp, L.grid, st); break;
      case 1: e = launch_prefill2_t<1, false>(tp, L.grid, st); break;
      default: e = launch_prefill2_t<2, false>(tp, L.grid, st); break;
    }
  }
  if (e != cudaSuccess) return -1;
  *name = "tc_prefill";
  return 1;
}

}  // namespace bsra
