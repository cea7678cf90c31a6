// tc_prefill2.cuh — ragged paged prefill on tcgen05 with two softmax warpgroups (T_q = 64/128).
//
// Same math and plan contract as tc_prefill.cuh (one work item = (request, kv head, q tile of
// 128 head-fused rows, kv chunk) from Algorithm 1, App. A head fusion, online softmax P:95,
// writethrough App. D.2), organised so that neither the tensor core nor the TMA engine waits on
// address arithmetic:
//   * the CTA's plan queue is split into two item streams (even / odd queue positions), one per
//     softmax warpgroup (WG); WG w owns S/P_w and O_w in TMEM (4 x 128 columns);
//   * a scheduler warp walks the two streams' KV tiles in a fixed interleaved order, batch-loads
//     the tiles' BSR page ids with all 32 lanes, and publishes one small descriptor per tile into
//     a shared-memory ring — the producers and the MMA warp only read descriptors;
//   * warp 0 loads Q (per WG) and K, warp 1 loads V through separate rings; per page one TMA box
//     {64 d, B_c tokens} per 64-column half, page id from the descriptor (§3.2.1);
//   * the MMA warp issues S_w = Q_w K^T as soon as K has landed and WG w is not holding its S
//     buffer, and O_w += P_w V with P_w read straight from TMEM (TS-MMA; P overwrites the
//     consumed S columns);
//   * softmax reads S from TMEM twice (max pass, exp pass) to keep registers low, ex2.approx with
//     the scale folded into an FFMA, lazy O rescale (threshold 2^8, exact).
// Ordering facts used: tcgen05 MMAs of one thread complete in issue order, so S_w(t+1) ready
// implies PV_w(t) done (O_w quiescent while WG w runs its softmax).
#pragma once
#include "tc_decode.cuh"
#include "tc_kernels.hpp"

namespace bsra {

namespace pre2 {
constexpr int kTile = 128;
// K ring depth 2 (not 3): the kernel's shared memory then stays under the 196 KB carve-out step
// and the SM keeps ~60 KB of L1; with a third K stage (224 KB, carve-out 228 KB) the same kernel
// measured 7 % slower (A/B on one box: 541 vs 575 us per configs[2] layer without o stores, and
// 8 KB of unused padding alone costs the same — the ring depth itself is not the limit).
#ifndef BSRA_PRE2_KSTAGES
#define BSRA_PRE2_KSTAGES 2
#endif
constexpr int kKStages = BSRA_PRE2_KSTAGES;
#ifndef BSRA_PRE2_VSTAGES
#define BSRA_PRE2_VSTAGES 2
#endif
constexpr int kVStages = BSRA_PRE2_VSTAGES;
constexpr int kDesc = 12;          // tile-descriptor ring
constexpr int kHalf = 128 * 128;   // 16 KB: 128 rows x 128 B
constexpr int kOp = 2 * kHalf;     // 32 KB operand (128 x 128 bf16, two SW128 halves)
constexpr int kOffQ = 0;           // [2 WGs]
constexpr int kOffK = 2 * kOp;
constexpr int kOffV = kOffK + kKStages * kOp;
constexpr int kOffBar = kOffV + kVStages * kOp;
constexpr int kOffDesc = kOffBar + 512;
#ifndef BSRA_PRE2_PAD
#define BSRA_PRE2_PAD 0
#endif
constexpr int kSmemBytes = kOffDesc + kDesc * 96 + 1024 + BSRA_PRE2_PAD;
constexpr int kThreads = 384;  // warps 0 Q+K producer, 1 V producer, 2 MMA, 3 scheduler, 4-7 WG0, 8-11 WG1
constexpr uint32_t kTmemCols = 512;  // S/P_w at w*128, O_w at 256 + w*128
constexpr float kRescaleThresh = 8.f;
#ifndef BSRA_PRE2_REGS_LOW
#define BSRA_PRE2_REGS_LOW 96
#endif
constexpr int kRegsLow = BSRA_PRE2_REGS_LOW;         // warpgroup 0 (producers, MMA, scheduler)
// The pool is what the CTA was launched with (168 per thread x 384 threads), not the SM's 64K:
// an inc the released registers cannot cover blocks forever.
constexpr int kRegsLaunch = 168;
// one-pass softmax (S held in registers, one TMEM read per tile) — needs the register split
#ifndef BSRA_PRE2_ONEPASS
#define BSRA_PRE2_ONEPASS 1
#endif
constexpr int kRegsHigh = (3 * kRegsLaunch - kRegsLow) / 2 / 8 * 8;  // each softmax warpgroup
static_assert(128 * kRegsLow + 256 * kRegsHigh <= 384 * kRegsLaunch, "register split exceeds the CTA's pool");
// exp2 split between the MUFU (4/clk/SMSP) and a cubic on the FMA pipes: kEmuPairs of every 8
// element pairs take the polynomial (FA4's exp2 emulation)
#ifndef BSRA_PRE2_EMU
#define BSRA_PRE2_EMU 0
#endif
constexpr int kEmuPairs = BSRA_PRE2_EMU;
}  // namespace pre2

// One KV tile of the interleaved order, as published by the scheduler warp.
struct TileDesc {
  int32_t w;           // softmax WG (-1: end of schedule)
  int32_t flags;       // bit0: first tile of its item, bit1: last tile of its item
  int32_t kvh;
  int32_t t0;          // first token of the tile within the request
  int32_t n;           // tokens in the tile
  int32_t head0, tok0; // Q tile coordinates (first tile only)
  int32_t pad;
  int32_t page[16];    // page id of sub-block j (B_c tokens, or 128 of a page >= 128)
};
static_assert(sizeof(TileDesc) == 96, "TileDesc layout");

// Walks one WG's item stream (queue positions it0+w, it0+w+2, ...) tile by tile.
struct ItemStream {
  int it, it1, stride;
  int ti;
  DecItem d;
  __device__ __forceinline__ void init(const PlanView& pv, int g, int first, int end, int step) {
    it = first;
    it1 = end;
    stride = step;
    ti = 0;
    skip_empty(pv, g);
  }
  __device__ __forceinline__ void skip_empty(const PlanView& pv, int g) {
    while (it < it1) {
      d = dec_item(pv, it, g);
      if (d.ntiles > 0) return;
      it += stride;
    }
  }
  __device__ __forceinline__ bool alive() const { return it < it1; }
  __device__ __forceinline__ void advance(const PlanView& pv, int g) {
    if (++ti < d.ntiles) return;
    ti = 0;
    it += stride;
    skip_empty(pv, g);
  }
};

// Deterministic interleave of the two streams: alternate while both are alive.
// (nstream = 1 only in the one-WG timing experiment: stream 1 is empty.)
struct Interleave {
  ItemStream s0, s1;
  int turn = 0;
  __device__ __forceinline__ void init(const PlanView& pv, int g, int it0, int it1, int nstream = 2) {
    s0.init(pv, g, it0, it1, nstream);
    s1.init(pv, g, nstream == 2 ? it0 + 1 : it1, it1, nstream);
    turn = 0;
  }
  __device__ __forceinline__ int pick() const {  // -1 when both exhausted
    if (s0.alive() && s1.alive()) return turn;
    if (s0.alive()) return 0;
    if (s1.alive()) return 1;
    return -1;
  }
  __device__ __forceinline__ void step(const PlanView& pv, int g, int w) {
    const bool both = s0.alive() && s1.alive();
    if (w == 0) s0.advance(pv, g);
    else s1.advance(pv, g);
    if (both) turn ^= 1;
  }
};

// kPair = false: T_q in {64, 128}; the two WGs run different items (two item streams).
// kPair = true:  T_q = 256; both WGs run the same item, WG w on fused rows [128w, 128w + 128), so
//                every K/V tile staged in smem feeds 256 query rows (half the L2->smem bytes per
//                flop of the streamed form, which the no-compute timing mode showed to be the bound).
// kVar: attention variants on (sliding window / soft-cap, read from p at run time); the default
// instantiation compiles them out so the plain path carries none of their per-tile work.
template <int kMask, bool kPair, bool kF16, bool kVar>
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
  uint64_t* desc_full = bar_o + 2;           // [kDesc] descriptor published
  uint64_t* desc_empty = desc_full + kDesc;  // [kDesc] released by K producer, V producer, MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(desc_empty + kDesc);
  TileDesc* descs = reinterpret_cast<TileDesc*>(smem + kOffDesc);

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
    for (int s = 0; s < kDesc; ++s) {
      ptx::mbar_init(&desc_full[s], 1);
      ptx::mbar_init(&desc_empty[s], 3);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();  // PDL: the next kernel's CTAs may take SMs this grid releases
  // register split (each role branch below): warpgroup 0 (producers, MMA issuer, scheduler)
  // gives registers to the two softmax warpgroups (128 x kRegsLow + 256 x kRegsHigh = 64K)
  const int B = tp.box_tok;
  // item streams: 2 (one per softmax WG); 1 when paired (both WGs on every item) or in the
  // one-WG timing experiment
#ifdef BSRA_EXPERIMENTS
  // timing experiments and the CTA-0 pipeline trace (scripts/trace_prefill.py); the shipped
  // build compiles them out (dbg = 0, no trace stores)
  const int dbg = tp.dbg;
  long long* const trace = (p.trace && blockIdx.x == 0) ? p.trace : nullptr;
#define BSRA_TRACE(ev, i) \
  if (trace && (i) < 1024) trace[(ev) * 1024 + (i)] = clock64();
  if (p.trace && threadIdx.x == 0) p.trace[16 * 1024 + blockIdx.x] = (long long)ptx::globaltimer_ns();
#else
  constexpr int dbg = 0;
#define BSRA_TRACE(ev, i)
#endif
  const int nstream = (kPair || (dbg & 4)) ? 1 : 2;
  const int ps = p.page_size;
  if (threadIdx.x == 0) BSRA_TRACE(9, 0);

  if (warp == 3) {
    ptx::setmaxnreg_dec<kRegsLow>();
    // ===================== scheduler: interleaved tile descriptors =====================
    Interleave il;
    il.init(pv, g, it0, it1, nstream);
    const int spp = kTile / B;             // sub-blocks of a full tile (<= 16)
    const int G = min(4, 32 / spp);        // positions per batched index load
    int pos = 0;
    bool done = false;
    while (!done) {
      // collect up to G positions (warp-uniform bookkeeping)
      int cw[4], cflags[4], ckvh[4], ct0[4], cn[4], chead0[4], ctok0[4];
      int64_t cpb[4];
      int cnt = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= G) break;
        const int w = il.pick();
        if (w < 0) {
          done = true;
          break;
        }
        const ItemStream& s = w == 0 ? il.s0 : il.s1;
        const DecItem& d = s.d;
        cw[k] = w;
        cflags[k] = (s.ti == 0 ? 1 : 0) | (s.ti + 1 == d.ntiles ? 2 : 0);
        ckvh[k] = d.kvh;
        ct0[k] = (int)(d.kb + (int64_t)s.ti * kTile);
        cn[k] = (int)imin64(kTile, d.ke - ct0[k]);
        chead0[k] = d.kvh * g + (g > 128 ? d.row0 % g : 0);
        ctok0[k] = (int)d.qo_begin + d.row0 / g;
        cpb[k] = d.page_begin;
        il.step(pv, g, w);
        cnt = k + 1;
      }
      // batched page-id loads: lane -> (position lane / spp, sub-block lane % spp)
      const int kq = lane / spp, j = lane % spp;
      int page = 0;
      if (kq < cnt) {
        int t0 = 0, n = 0;
        int64_t pb = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k == kq) {
            t0 = ct0[k];
            n = cn[k];
            pb = cpb[k];
          }
        // paged: the sub-block's page id; contiguous KV: its token coordinate
        if (j * B < n) page = p.kv_ragged ? (int)(pb + t0 + j * B) : __ldg(p.page_indices + pb + (t0 + j * B) / ps);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= cnt) break;
        const int slot = pos % kDesc;
        const uint32_t ph = ((pos / kDesc) & 1) ^ 1;
        ptx::mbar_wait(&desc_empty[slot], ph);
        TileDesc& D = descs[slot];
        if (lane == 0) {
          D.w = cw[k];
          D.flags = cflags[k];
          D.kvh = ckvh[k];
          D.t0 = ct0[k];
          D.n = cn[k];
          D.head0 = chead0[k];
          D.tok0 = ctok0[k];
        }
        if (kq == k) D.page[j] = page;
        // bar.sync (not __syncwarp): orders every lane's descriptor writes before lane 0's arrive
        // in a form compute-sanitizer's racecheck tracks through the mbarrier hand-off
        ptx::named_bar_sync(6, 32);
        if (lane == 0) ptx::mbar_arrive(&desc_full[slot]);
        if (lane == 0) BSRA_TRACE(10, pos);
        ++pos;
      }
    }
    // terminator
    const int slot = pos % kDesc;
    ptx::mbar_wait(&desc_empty[slot], ((pos / kDesc) & 1) ^ 1);
    if (lane == 0) {
      descs[slot].w = -1;
      ptx::mbar_arrive(&desc_full[slot]);
    }
  } else if (warp == 0 || warp == 1) {
    ptx::setmaxnreg_dec<kRegsLow>();
    // ===================== producers: warp 0 = Q + K, warp 1 = V =====================
    const bool isK = warp == 0;
    if (lane == 0) {
      if (isK) ptx::tma_prefetch_desc(&tp.tq);
      ptx::tma_prefetch_desc(isK ? &tp.tk : &tp.tv);
    }
    uint32_t qphase = 3;  // bit w: phase of empty_q[w] to wait for (first wait passes)
    int stage = 0;
    uint32_t ephase = 1;
    const int nst = isK ? kKStages : kVStages;
    uint64_t* fullx = isK ? full_k : full_v;
    uint64_t* emptyx = isK ? empty_k : empty_v;
    const CUtensorMap* tm = isK ? &tp.tk : &tp.tv;
    const int ring = isK ? kOffK : kOffV;
    for (int pos = 0;; ++pos) {
      const int slot = pos % kDesc;
      ptx::mbar_wait(&desc_full[slot], (pos / kDesc) & 1);
      const TileDesc& D = descs[slot];
      if (D.w < 0) break;
      const int kvh = D.kvh, t0 = D.t0, n = D.n;
      const int nsub = (n + B - 1) / B;
      const int pg = lane < nsub ? D.page[lane] : 0;
      // tiles start page-aligned (chunk alignment is a multiple of B), so sub-blocks of pages
      // <= 128 tokens start at slot 0; only pages > 128 tokens need the in-page offset.
      // Contiguous KV: the descriptor holds the token coordinate, the page coordinate is 0.
      const int off = p.kv_ragged ? pg : ps <= kTile ? 0 : (t0 + lane * B) % ps;
      const int page = p.kv_ragged ? 0 : pg;
      if (isK && (D.flags & 1) && lane == 0) {  // Q of the item's WG (paired: both halves)
        const int w = kPair ? 0 : D.w;
        for (int h = 0; h < (kPair ? 2 : 1); ++h) {
          const int wb = w + h;
          ptx::mbar_wait(&empty_q[wb], (qphase >> wb) & 1);
          ptx::mbar_arrive_expect_tx(&full_q[wb], kOp);
          uint8_t* qdst = smem + kOffQ + wb * kOp;
          const int tok = D.tok0 + h * (128 / g);  // rows [128h, 128h + 128): g <= 128 divides 128
          ptx::tma_load_3d(qdst, &tp.tq, &full_q[wb], 0, D.head0, tok);
          ptx::tma_load_3d(qdst + kHalf, &tp.tq, &full_q[wb], 64, D.head0, tok);
        }
      }
      if (isK && (D.flags & 1)) qphase ^= kPair ? 3u : (1u << D.w);
      ptx::named_bar_sync(3 + warp, 32);  // every lane's descriptor reads precede the release
      if (lane == 0) ptx::mbar_arrive(&desc_empty[slot]);  // descriptor fields are in registers
      if (lane == 0) {
        ptx::mbar_wait(&emptyx[stage], ephase);
        ptx::mbar_arrive_expect_tx(&fullx[stage], (uint32_t)nsub * B * 256);
      }
      __syncwarp();
      if (lane < nsub) {
        uint8_t* dst = smem + ring + stage * kOp + lane * B * 128;
        if (lane == 0) BSRA_TRACE(isK ? 0 : 1, pos);
        ptx::tma_load_4d(dst, tm, &fullx[stage], 0, kvh, off, page);
        ptx::tma_load_4d(dst + kHalf, tm, &fullx[stage], 64, kvh, off, page);
      }
      __syncwarp();
      if ((dbg & 8) && lane == 0) {  // timing experiment: TMA issue -> landed latency
        ptx::mbar_wait(&fullx[stage], ephase ^ 1);
        BSRA_TRACE(isK ? 15 : 14, pos);
      }
      __syncwarp();
      if (++stage == nst) {
        stage = 0;
        ephase ^= 1;
      }
    }
  } else if (warp == 2) {
    ptx::setmaxnreg_dec<kRegsLow>();
    // ===================== MMA issuer =====================
    const uint32_t fmt = tp.f16 ? 0u : 1u;
    const uint32_t idS = ptx::idesc_f16(fmt, 128, kTile, 0, 0);  // A = Q (K-major), B = K (K-major)
    const uint32_t idO = ptx::idesc_f16(fmt, 128, 128, 0, 1);    // A = P (TMEM), B = V (MN-major)
    const uint32_t sbase = ptx::smem_u32(smem);
    // S_w = Q_w K^T from K stage ks; descriptors +2 (32 B) per K step inside a 64-column atom,
    // +1024 (16 KB) per atom
    auto issue_s = [&](int w, int ks) {
      const uint64_t a0 = ptx::smem_desc_sw128(sbase + kOffQ + w * kOp, 16, 1024);
      const uint64_t b0 = ptx::smem_desc_sw128(sbase + kOffK + ks * kOp, 16, 1024);
      const uint32_t dS = tmem + w * 128;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t step = (uint64_t)((kk >> 2) * (kHalf >> 4) + (kk & 3) * 2);
        if (!(dbg & 2)) ptx::mma_f16_ss_warp(dS, a0 + step, b0 + step, idS, kk > 0);
      }
    };
    // O_w += P_w V from V stage vs; +128 (2 KB = 16 tokens) per K step of the MN-major V
    auto issue_pv = [&](int w, int vs, bool first) {
      const uint64_t b0 = ptx::smem_desc_sw128(sbase + kOffV + vs * kOp, kHalf, 1024);
      const uint32_t dO = tmem + 256 + w * 128, aP = tmem + w * 128;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        if (!(dbg & 2)) ptx::mma_f16_ts_warp(dO, aP + kk * 8, b0 + (uint64_t)(kk * 128), idO, (first && kk == 0) ? 0u : 1u);
    };
    // rows past the chunk end -> 0 in the V stage (0 * garbage could be NaN)
    auto zero_v_tail = [&](int vs, int n) {
      uint8_t* vS = smem + kOffV + vs * kOp;
      for (int rr = n + lane; rr < kTile; rr += 32) {
        uint4* v0 = reinterpret_cast<uint4*>(vS + rr * 128);
        uint4* v1 = reinterpret_cast<uint4*>(vS + kHalf + rr * 128);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          v0[jj] = make_uint4(0, 0, 0, 0);
          v1[jj] = make_uint4(0, 0, 0, 0);
        }
      }
      ptx::fence_proxy_async();
      __syncwarp();
    };
    if constexpr (kPair) {
      // Both WGs on every tile t, issued as  S0(t) S1(t) | PV0(t) S0(t+1) PV1(t) S1(t+1) | ...
      // S_w(t+1) overwrites the columns P_w(t) occupies, so it is issued after PV_w(t) (the tensor
      // pipe executes one thread's MMAs in order); WG1's softmax of t overlaps PV0(t), S0(t+1).
      int kst = 0, vst = 0;
      uint32_t kph = 0, vph = 0, qph = 0, pph[2] = {0, 0};
      int pos = 0;
      const TileDesc* D = &descs[0];
      ptx::mbar_wait(&desc_full[0], 0);
      bool have = D->w >= 0;
      int flags = have ? D->flags : 0, n = have ? D->n : 0;
      int pos_s = 0;  // trace index of the S being issued
      auto s_pair_half = [&](int w, int fl) {  // S_w of the tile in K stage kst
        if (fl & 1) ptx::mbar_wait(&full_q[w], qph);
        if (lane == 0 && w == 0) BSRA_TRACE(13, pos_s);
        if (w == 0) ptx::mbar_wait(&full_k[kst], kph);
        if (lane == 0 && w == 0) BSRA_TRACE(2, pos_s);
        ptx::tc_fence_after();
        issue_s(w, kst);
        ptx::mma_commit_warp(&bar_s[w]);
        if (fl & 2) ptx::mma_commit_warp(&empty_q[w]);  // the item's last S: Q_w buffer free
        if (w == 1) {
          ++pos_s;
          ptx::mma_commit_warp(&empty_k[kst]);
          if (fl & 1) qph ^= 1;
          if (++kst == kKStages) {
            kst = 0;
            kph ^= 1;
          }
        }
      };
      if (have) {
        s_pair_half(0, flags);
        s_pair_half(1, flags);
      }
      while (have) {
        const int slot = pos % kDesc;
        if (lane == 0) BSRA_TRACE(3, pos);
        ptx::mbar_wait(&full_v[vst], vph);
        if (n < kTile) zero_v_tail(vst, n);
        ptx::mbar_wait(&p_ready[0], pph[0]);
        pph[0] ^= 1;
        ptx::tc_fence_after();
        issue_pv(0, vst, flags & 1);
        if (flags & 2) ptx::mma_commit_warp(&bar_o[0]);
        // next tile's descriptor (the scheduler runs ahead)
        const int npos = pos + 1, nslot = npos % kDesc;
        ptx::mbar_wait(&desc_full[nslot], (npos / kDesc) & 1);
        const TileDesc* N = &descs[nslot];
        const bool nhave = N->w >= 0;
        const int nflags = nhave ? N->flags : 0, nn = nhave ? N->n : 0;
        if (nhave) s_pair_half(0, nflags);
        ptx::mbar_wait(&p_ready[1], pph[1]);
        pph[1] ^= 1;
        ptx::tc_fence_after();
        issue_pv(1, vst, flags & 1);
        ptx::mma_commit_warp(&empty_v[vst]);
        if (flags & 2) ptx::mma_commit_warp(&bar_o[1]);
        ptx::named_bar_sync(5, 32);  // all lanes' descriptor reads precede the release
        ptx::mbar_arrive_warp(&desc_empty[slot]);
        if (++vst == kVStages) {
          vst = 0;
          vph ^= 1;
        }
        if (nhave) s_pair_half(1, nflags);
        pos = npos;
        have = nhave;
        flags = nflags;
        n = nn;
      }
    } else {
      // Streamed: two cursors over the descriptor ring, S in order (K ring) and PV in order (V
      // ring). A WG has one S buffer, so its next S is issued only after the PV of its current
      // tile (in-order tensor pipe => no WAR hazard on TMEM).
      int kst = 0, vst = 0;
      uint32_t kph = 0, vph = 0;
      // per-WG phase bits and the "S buffer held" flags as bitmasks (register-resident; arrays
      // indexed by the runtime WG would live in local memory on the issue path)
      uint32_t qph = 0, pph = 0, pending = 0;
      int s_pos = 0, pv_pos = 0;
      bool s_done = false;
      for (;;) {
        // ---- issue S in order while the next tile's WG is not holding its S buffer
        while (!s_done) {
          const int slot = s_pos % kDesc;
          const uint32_t ph = (s_pos / kDesc) & 1;
          if (pv_pos == s_pos) ptx::mbar_wait(&desc_full[slot], ph);
          else if (!ptx::mbar_test_wait_warp(&desc_full[slot], ph)) break;
          const TileDesc& D = descs[slot];
          const int w = D.w;
          if (w < 0) {
            s_done = true;
            break;
          }
          if ((pending >> w) & 1) break;
          const int flags = D.flags;
          if (flags & 1) {  // first tile of an item: its Q must have landed
            ptx::mbar_wait(&full_q[w], (qph >> w) & 1);
            qph ^= 1u << w;
          }
          ptx::mbar_wait(&full_k[kst], kph);
          if (lane == 0) BSRA_TRACE(2, s_pos);
          ptx::tc_fence_after();
          issue_s(w, kst);
          ptx::mma_commit_warp(&empty_k[kst]);
          ptx::mma_commit_warp(&bar_s[w]);
          if (flags & 2) ptx::mma_commit_warp(&empty_q[w]);  // last S of the item: Q buffer free
          if (++kst == kKStages) {
            kst = 0;
            kph ^= 1;
          }
          pending |= 1u << w;
          ++s_pos;
        }
        if (pv_pos == s_pos) break;  // schedule finished and every PV issued
        // ---- PV of the oldest tile
        const int slot = pv_pos % kDesc;
        const TileDesc& D = descs[slot];
        const int w = D.w, n = D.n, flags = D.flags;
        ptx::mbar_wait(&full_v[vst], vph);
        if (n < kTile) zero_v_tail(vst, n);
        ptx::mbar_wait(&p_ready[w], (pph >> w) & 1);
        pph ^= 1u << w;
        if (lane == 0) BSRA_TRACE(3, pv_pos);
        ptx::tc_fence_after();
        issue_pv(w, vst, flags & 1);
        ptx::mma_commit_warp(&empty_v[vst]);
        if (flags & 2) ptx::mma_commit_warp(&bar_o[w]);
        ptx::named_bar_sync(5, 32);  // all lanes' descriptor reads precede the release
        ptx::mbar_arrive_warp(&desc_empty[slot]);
        if (++vst == kVStages) {
          vst = 0;
          vph ^= 1;
        }
        pending &= ~(1u << w);
        ++pv_pos;
      }
    }
  } else if (warp >= 4) {
    ptx::setmaxnreg_inc<kRegsHigh>();
    // ===================== softmax warpgroups =====================
    const int w = (warp - 4) >> 2;        // WG index
    const int q4 = warp & 3;              // TMEM lane quarter
    const int r = q4 * 32 + lane;         // fused row of the tile
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_addr + w * 128;
    const uint32_t tO = tmem + lane_addr + 256 + w * 128;
    const float sc = p.scale_log2;
    uint32_t sph = 0, oph = 0;
    int tcount = 0;
    const int ri = kPair ? w * 128 + r : r;  // this thread's row within the item
    const int first_it = kPair ? it0 : it0 + w;
    for (int it = first_it; (kPair || w < nstream) && it < it1; it += nstream) {
      const DecItem d = dec_item(pv, it, g);
      if (r == 0 && w == 0) BSRA_TRACE(14, it - it0);
      const bool row_ok = ri < d.nrows;
      const int f = d.row0 + ri;
      const int tok = f / g, head = d.kvh * g + f % g;
      const int64_t lim = kMask == 1 ? d.lk - d.lq + tok : d.ke - 1;
      const int64_t mbase = kMask == 2 ? p.mask_indptr[d.req] + (int64_t)tok * d.lk : 0;
      // variants: sliding-window lower bound of this row (R26), soft-cap (R27) — both go through
      // the general (per-element) path; plain tiles keep the fast path
      const int64_t wlo = kVar && p.window > 0 ? d.lk - d.lq + tok - p.window + 1 : INT64_MIN / 2;
      const bool capped = kVar && p.soft_cap > 0.f;
      // ALiBi (R30): raw-unit bias aslope * (t - apos) on every element, after the soft-cap
      const bool biased = kVar && p.alibi;
      const float aslope = biased ? alibi_slope_raw(p, head) : 0.f;
      const float apos = (float)(d.lk - d.lq + tok);
      float m = -INFINITY, l = 0.f;
      for (int ti = 0; ti < d.ntiles; ++ti) {
        const int64_t t0 = d.kb + (int64_t)ti * kTile;
        const int n = (int)imin64(kTile, d.ke - t0);
        const int64_t vis_end = row_ok ? (kMask == 1 ? imin64(lim + 1, t0 + n) : t0 + n) : t0;
        const int nvis = (int)(vis_end > t0 ? vis_end - t0 : 0);
        const int vbeg = kVar && wlo > t0 ? (int)imin64(wlo - t0, kTile) : 0;  // first visible column
        const bool need_mask = kMask == 2 || nvis < kTile || vbeg > 0 || capped || biased;
        const float abase = aslope * ((float)t0 - apos);  // bias of column 0 of this tile
        ptx::mbar_wait(&bar_s[w], sph);
        sph ^= 1;
        if (r == 0) BSRA_TRACE(5 + 2 * w, tcount);
        ptx::tc_fence_after();
        if (dbg & 1) {  // timing experiment: no softmax work (results are garbage)
          ptx::tc_fence_before();
          ptx::mbar_arrive(&p_ready[w]);
          ++tcount;
          continue;
        }
        // the variant instantiation keeps the two-pass form (the soft-cap needs the registers)
        constexpr bool kOnePass = BSRA_PRE2_ONEPASS && !kVar;
        if constexpr (kOnePass) {
        // ---- one pass (registers from setmaxnreg): all 128 S columns in one TMEM round trip,
        // mask / soft-cap, row max, P = 2^(s*scale - m) packed to 16-bit pairs over the consumed
        // S columns; the rare O rescale goes after P (O_w is quiescent until p_ready)
        float s[128];
        ptx::tmem_ld32(tS, s);
        ptx::tmem_ld32(tS + 32, s + 32);
        ptx::tmem_ld32(tS + 64, s + 64);
        ptx::tmem_ld32(tS + 96, s + 96);
        ptx::tmem_ld_wait();
        if (need_mask) {
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            bool vis = j < nvis && j >= vbeg;
            if (kMask == 2) vis = vis && mask_bit(p.mask, mbase + t0 + j);
            s[j] = vis ? (capped ? soft_cap_raw(p, s[j]) : s[j]) : -INFINITY;
          }
        }
        float a0 = fmaxf(s[0], s[1]), a1 = fmaxf(s[2], s[3]), a2 = fmaxf(s[4], s[5]), a3 = fmaxf(s[6], s[7]);
#pragma unroll
        for (int j = 8; j < 128; j += 4) {
          a0 = fmaxf(a0, s[j]);
          a1 = fmaxf(a1, s[j + 1]);
          a2 = fmaxf(a2, s[j + 2]);
          a3 = fmaxf(a3, s[j + 3]);
        }
        const float mt = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)) * sc;
        float alpha = 1.f;
        bool rescale = false;
        if (mt > m + kRescaleThresh) {
          if (m != -INFINITY) {
            alpha = ptx_ex2(m - mt);
            rescale = true;
          }
          m = mt;
        }
        const float mneg = m == -INFINITY ? 0.f : -m;
        const float2 sc2 = make_float2(sc, sc), mn2 = make_float2(mneg, mneg);
        const float2 mn2h = make_float2(mneg - 0.5f, mneg - 0.5f);  // poly_ex2x2_shifted takes x - 1/2
        float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float2 x;
            const float2 sv = make_float2(s[c * 32 + j], s[c * 32 + j + 1]);
            if (((j >> 1) & 7) < kEmuPairs) {  // kEmuPairs of every 8 pairs on the FMA pipes
              x = poly_ex2x2_shifted(__ffma2_rn(sv, sc2, mn2h));
            } else {
              x = __ffma2_rn(sv, sc2, mn2);
              x.x = ptx_ex2(x.x);
              x.y = ptx_ex2(x.y);
            }
            rs[(j >> 1) & 3] = __fadd2_rn(rs[(j >> 1) & 3], x);
            if constexpr (kF16) {
              __half2 h = __floats2half2_rn(x.x, x.y);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(x.x, x.y);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          ptx::tmem_st16(tS + c * 16, pk);
        }
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
        const float2 r01 = __fadd2_rn(rs[0], rs[1]), r23 = __fadd2_rn(rs[2], rs[3]);
        l = l * alpha + ((r01.x + r01.y) + (r23.x + r23.y));
        } else {
        // ---- pass 1: raw row max (two 32-column TMEM loads in flight per round trip)
        float mx = (dbg & 16) ? 0.f : -INFINITY;  // dbg 16: timing experiment, no max pass
#pragma unroll
        for (int c = 0; c < ((dbg & 16) ? 0 : 4); c += 2) {
          float s[64];
          ptx::tmem_ld32(tS + c * 32, s);
          ptx::tmem_ld32(tS + c * 32 + 32, s + 32);
          ptx::tmem_ld_wait();
          if (need_mask) {
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              bool vis = c * 32 + j < nvis && c * 32 + j >= vbeg;
              if (kMask == 2) vis = vis && mask_bit(p.mask, mbase + t0 + c * 32 + j);
              float x = s[j];
              if (biased) x = (capped ? soft_cap_raw(p, x) : x) + fmaf(aslope, (float)(c * 32 + j), abase);
              s[j] = vis ? x : -INFINITY;
            }
          }
          float a0 = fmaxf(s[0], s[1]), a1 = fmaxf(s[2], s[3]), a2 = fmaxf(s[4], s[5]), a3 = fmaxf(s[6], s[7]);
#pragma unroll
          for (int j = 8; j < 64; j += 4) {
            a0 = fmaxf(a0, s[j]);
            a1 = fmaxf(a1, s[j + 1]);
            a2 = fmaxf(a2, s[j + 2]);
            a3 = fmaxf(a3, s[j + 3]);
          }
          mx = fmaxf(mx, fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
        }
        // soft-cap is monotone, so the capped max is the cap of the raw max (-inf stays -inf)
        const float mt = (capped && !biased && mx != -INFINITY ? soft_cap_raw(p, mx) : mx) * sc;
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
        // packed fp32 pairs (FFMA2 / FADD2) for the scale and the row sum; four independent sums
        const float mneg = m == -INFINITY ? 0.f : -m;
        const float2 sc2 = make_float2(sc, sc), mn2 = make_float2(mneg, mneg);
        const float2 mn2h = make_float2(mneg - 0.5f, mneg - 0.5f);  // poly_ex2x2_shifted takes x - 1/2
        float2 rs[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float sbuf[2][32];  // chunk c+1's TMEM load overlaps chunk c's exponentials
        ptx::tmem_ld32(tS, sbuf[0]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float* s = sbuf[c & 1];
          if (c + 1 < 4) ptx::tmem_ld32(tS + (c + 1) * 32, sbuf[(c + 1) & 1]);
          if (need_mask) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              bool vis = c * 32 + j < nvis && c * 32 + j >= vbeg;
              if (kMask == 2) vis = vis && mask_bit(p.mask, mbase + t0 + c * 32 + j);
              float x = capped ? soft_cap_raw(p, s[j]) : s[j];
              if (biased) x += fmaf(aslope, (float)(c * 32 + j), abase);
              s[j] = vis ? x : -INFINITY;
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float2 x;
            if (((j >> 1) & 7) < kEmuPairs) {  // kEmuPairs of every 8 pairs on the FMA pipes
              x = poly_ex2x2_shifted(__ffma2_rn(make_float2(s[j], s[j + 1]), sc2, mn2h));
            } else {
              x = __ffma2_rn(make_float2(s[j], s[j + 1]), sc2, mn2);
              x.x = ptx_ex2(x.x);
              x.y = ptx_ex2(x.y);
            }
            rs[(j >> 1) & 3] = __fadd2_rn(rs[(j >> 1) & 3], x);
            if constexpr (kF16) {
              __half2 h = __floats2half2_rn(x.x, x.y);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            } else {
              __nv_bfloat162 h = __floats2bfloat162_rn(x.x, x.y);
              pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            }
          }
          ptx::tmem_st16(tS + c * 16, pk);
          ptx::tmem_ld_wait();  // chunk c+1 has landed (its columns are >= 32(c+1) > P's 16(c+1))
        }
        const float2 r01 = __fadd2_rn(rs[0], rs[1]), r23 = __fadd2_rn(rs[2], rs[3]);
        l = l * alpha + ((r01.x + r01.y) + (r23.x + r23.y));
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_ready[w]);
        if (r == 0) BSRA_TRACE(6 + 2 * w, tcount);
        ++tcount;
      }
      pdl_wait();  // PDL: the previous kernel on the stream has completed before we write
      // ---- epilogue: wait for the item's last PV, normalise, write
      if (r == 0 && w == 0) BSRA_TRACE(11, it - it0);
      if (d.ntiles > 0) {
        ptx::mbar_wait(&bar_o[w], oph);
        oph ^= 1;
        ptx::tc_fence_after();
      }
      if (r == 0 && w == 0) BSRA_TRACE(12, it - it0);
      const bool empty_row = !(l > 0.f);
      const float inv = empty_row ? 0.f : p.v_scale / l;  // v_scale: fp8 KV (R28), else 1
      const float lse = empty_row ? -INFINITY : (m + __log2f(l)) * kLn2;
      const int64_t orow = (d.qo_begin + tok) * p.H_qo + head;
      const int64_t prow = (int64_t)d.slot * p.T_slot + ri;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        float ov[32];
        if (d.ntiles > 0 && !(dbg & 128)) {  // dbg 128: timing experiment, no O read
          ptx::tmem_ld32(tO + c0, ov);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) ov[j] = 0.f;
        }
        if (!row_ok || (dbg & 64)) continue;  // dbg 64: timing experiment, no o stores
        // 256-bit stores: a lane writes whole 32-byte sectors of its row (half the instructions of
        // 16-byte stores; rows of a warp are scattered, so the instruction count is the cost)
        if (d.slot >= 0 || p.o_f32) {
          float* dstf = d.slot >= 0 ? p.part_o + prow * 128 + c0 : reinterpret_cast<float*>(p.o) + orow * 128 + c0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t wv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) wv[e] = __float_as_uint(ov[8 * j + e] * inv);
            ptx::st_global_v8(dstf + 8 * j, wv);
          }
        } else {
          uint16_t* dsth = reinterpret_cast<uint16_t*>(p.o) + orow * 128 + c0;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            uint32_t wv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float a0 = ov[16 * j + 2 * e] * inv, a1 = ov[16 * j + 2 * e + 1] * inv;
              if constexpr (kF16) {
                __half2 h = __floats2half2_rn(a0, a1);
                wv[e] = *reinterpret_cast<uint32_t*>(&h);
              } else {
                __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
                wv[e] = *reinterpret_cast<uint32_t*>(&h);
              }
            }
            ptx::st_global_v8(dsth + 16 * j, wv);
          }
        }
      }
      if (row_ok) {
        if (d.slot >= 0) p.part_lse[prow] = lse;
        else if (p.lse) p.lse[orow] = lse;
      }
      if (!kPair && d.slot >= 0 && p.fused_merge) {  // split item: the WG completing its merge list folds it
        volatile int* s_flag = reinterpret_cast<volatile int*>(tmem_slot + 1 + w);
        if constexpr (kF16) fused_contraction<__half, 128>(p, pv, d.slot, r, 128, 2 + w, s_flag);
        else fused_contraction<__nv_bfloat16, 128>(p, pv, d.slot, r, 128, 2 + w, s_flag);
      }
      ptx::tc_fence_before();  // O_w reads done before this WG's next p_ready (next item's PV)
      if (r == 0 && w == 0) BSRA_TRACE(4, it - it0);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) BSRA_TRACE(9, 1);
#ifdef BSRA_EXPERIMENTS
  if (p.trace && threadIdx.x == 0) p.trace[17 * 1024 + blockIdx.x] = (long long)ptx::globaltimer_ns();
#endif
#undef BSRA_TRACE
  if (warp == 2) ptx::tmem_dealloc<kTmemCols>(tmem);
}

template <int kMask, bool kPair, bool kF16, bool kVar>
inline cudaError_t launch_prefill2_f(const TcParams& tp, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_prefill2_kernel<kMask, kPair, kF16, kVar>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, pre2::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_tc(tc_prefill2_kernel<kMask, kPair, kF16, kVar>, grid, pre2::kThreads, pre2::kSmemBytes, st, tp);
}

template <int kMask, bool kPair, bool kF16>
inline cudaError_t launch_prefill2_v(const TcParams& tp, int grid, cudaStream_t st) {
  const bool var = tp.p.window > 0 || tp.p.soft_cap > 0.f || tp.p.alibi;
  return var ? launch_prefill2_f<kMask, kPair, kF16, true>(tp, grid, st)
             : launch_prefill2_f<kMask, kPair, kF16, false>(tp, grid, st);
}

template <int kMask, bool kPair>
inline cudaError_t launch_prefill2_t(const TcParams& tp, int grid, cudaStream_t st) {
  return tp.f16 ? launch_prefill2_v<kMask, kPair, true>(tp, grid, st) : launch_prefill2_v<kMask, kPair, false>(tp, grid, st);
}

}  // namespace bsra
