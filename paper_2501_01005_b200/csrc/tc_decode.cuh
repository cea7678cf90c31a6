// tc_decode.cuh — paged decode attention on tcgen05 tensor cores (T_q = 16 head-fused rows).
//
// Head-group fusion (App. A): the <= 16 fused rows of one (request, kv head, q tile)
// share every K/V byte. With so few rows the contraction is turned around ("swap-AB") so that
// the 128 KV tokens of a tile fill the MMA's M dimension:
//     S^T[128 tok x 16] = K[128 x D] . Q^T[D x 16]           (tcgen05, fp32 accumulate in TMEM)
//     O^T[D x 16]      += V^T[D x 128] . P^T[128 x 16]       (V^T is an MN-major view of V in smem)
// so one KV load serves all fused rows and the tensor core does the arithmetic while the kernel
// streams HBM (decode is HBM-bound, fig:varlen).
//
// Warp roles (one CTA per SM, persistent over the CTA's plan queue; warp 5 issues the MMAs):
//   warp 0      TMA producer (Q, K): per page one box of the 5-D pool view (d_lo, token_lo, half,
//               token_hi, page * cs + head) — both 64-column halves, group-major tiles (kGrp) —
//               or, half-major, one box {64 d, B_c tokens} per page and half of the 4-D view
//               (d, kv head, slot, page); the BSR `indices` give the page coordinate (the sparse
//               gather of §3.2.1, done by TMA). Runs ahead across items through a
//               kStages-deep smem ring.
//   warp 18     (fused-RoPE variant) the V producer
//   warps 10-12 more TMA producers (plain variant): warp 10 issues the V boxes; the row-gather
//   (10-16)     variant has 8 producer warps (0, 10..16), each issuing one K / V x column-half
//               quarter of half the tile's rows — TMA issue is serialised per warp
//               (scripts/tma_issue_bench.cu).
//   warps 1..4  128 threads: thread = TMEM lane = token (softmax) = head-dim row d (output).
//   warps 6..9  epilogue: O^T is double-buffered in TMEM (cols 32 / 48 by item parity); the
//               softmax warps hand each finished item over (row-sum partials + running max in
//               smem) and go on with the next one while these warps normalise and store o / lse
//               (and run the fused contraction for split items).
//   warp 5      MMA issuer: S^T(t) as soon as K(t) landed and the S^T buffer was read, PV(t-1)
//               once P(t-1) is written (s_free / p_full / o_free barriers), so the ~35-cycle
//               per-instruction MMA issue stays off the softmax chain. Online softmax in the log2 domain with
//               lazy rescaling: O^T accumulates in TMEM across tiles and is rescaled only when a
//               row max grows by more than 2^8 (the final o = O/l and lse use the same max, so the
//               result is exact). S^T and P^T are double-buffered and the next tile's S MMA is
//               issued before this tile's softmax when its K has landed.
// kC = live fused columns (4, 8 or 16) — only those run through the softmax; kMask = mask mode.
// Epilogue: unsplit rows write o / lse (writethrough, App. D.2), split rows fp32 partials.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "merge.cuh"
#include "ptx.cuh"

namespace bsra {

struct TcParams {
  AttnParams p;
  CUtensorMap tq;  // q  [N, H_qo, D]: dims (D, H_qo, N), box (64, q_hb, q_tb), SW128
  CUtensorMap tk;  // K pool: dims (D, H_kv, page_size, pages), box (64, 1, box_tok, 1), SW128
  CUtensorMap tv;  // V pool: same
  int32_t box_tok;  // min(page_size, 128)
  int32_t q_hb, q_tb;
  int32_t f16;      // 1 = fp16 inputs, 0 = bf16
  int32_t pdl;      // launched with programmatic dependent launch (host-side launch choice)
  int32_t cp;       // decode K/V gather: 0 = TMA boxes per page, 1 = 16-byte cp.async rows, 2 = TMA gather4 rows
  int64_t row_s0, row_s1, row_s2;  // gather4: (page, slot, head) strides in rows of the 2-D [rows, D] view
  int32_t grp;      // 1: page boxes of the 5-D pool view (both 64-column halves per box), group-major tiles
  int32_t cs;       // grp: pool page stride / head stride (the 5-D view's (page, head) coordinate = page * cs + head)
  int32_t dbg;      // BSRA_EXPERIMENTS builds only ($BSRA_DEBUG_PREFILL timing modes); 0 otherwise
};

// Kernel launch honouring TcParams::pdl (cudaLaunchAttributeProgrammaticStreamSerialization).
template <typename Kern>
inline cudaError_t launch_tc(Kern kernel, int grid, int threads, int smem, cudaStream_t st, const TcParams& tp) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = tp.pdl ? attr : nullptr;
  cfg.numAttrs = tp.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, tp);
}

// PDL device side: let the next kernel on the stream start launching, and before this kernel's
// first global write wait for the previous kernel to complete (no-ops without PDL).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

namespace dec {
constexpr int kTile = 128;         // tokens per KV tile (= MMA M)
constexpr int kN = 16;             // fused rows per tile (= MMA N)
constexpr int kStages = 3;
constexpr int kHalfBytes = kTile * 128;      // 128 tokens x 64 d x 2 B = 16 KB
constexpr int kKVBytes = 2 * kHalfBytes;     // one of K or V: 32 KB
constexpr int kStageBytes = 2 * kKVBytes;    // K + V: 64 KB
constexpr int kQBytes = 2 * kN * 128;        // 2 halves x 16 rows x 128 B = 4 KB
constexpr int kPBytes = 2 * kN * 128;        // P^T: 2 token-halves x 16 rows x 128 B
constexpr int kOffQ = kStages * kStageBytes;
constexpr int kOffP = kOffQ + 2 * kQBytes;   // two P^T buffers
constexpr int kOffBar = kOffP + 2 * kPBytes;
constexpr int kOffRed = kOffBar + 512;
// red [4][kN], vote flags [2][4], epilogue hand-off sums [2][4][kN] and max [2][kN]
constexpr int kOffItems = kOffRed + 1024;
constexpr int kStagedItems = 64;  // the CTA's first queue entries, decoded once into shared memory
constexpr int kOffMeta = kOffItems + kStagedItems * 80;  // merge-list metadata of staged split items
constexpr int kSmemBytes = kOffMeta + kStagedItems * 32 + 1024;  // + alignment slack
constexpr int kThreads = 320;  // producer, 4 softmax warps, MMA warp, 4 epilogue warps
#ifndef BSRA_ROPE_PRODUCERS
#define BSRA_ROPE_PRODUCERS 2
#endif
// + 8 RoPE warps (two per SM sub-partition) in the fused-RoPE variant, and (2 producers) warp 18
// issuing the V boxes
constexpr int kThreadsRope = 576 + 32 * (BSRA_ROPE_PRODUCERS - 1);
// Plain variant: + 3 producer warps (10..12). TMA issue is per-warp serialised (~65-160 cycles per
// instruction whatever the box size, and it scales with the number of issuing warps:
// scripts/tma_issue_bench.cu), so K and V boxes (and the four gather4 quarters) come from
// different warps.
constexpr int kThreadsPlain = kThreads + 96;
constexpr int kThreadsRow = kThreads + 224;  // row gather: 8 producer warps (0, 10..16)
constexpr int threads_for(bool rope, bool row = false) { return rope ? kThreadsRope : row ? kThreadsRow : kThreadsPlain; }
constexpr uint32_t kTmemCols = 64;  // S^T buffers at cols 0 / 16, O^T double buffer at 32 / 48
constexpr float kRescaleThresh = 8.f;  // log2 units: rescale O only when the max grows by > 2^8
}  // namespace dec

struct DecItem {
  int req, kvh, row0, nrows, slot, lq;
  int64_t kb, ke, lk, qo_begin, page_begin;
  int ntiles;
};

static_assert(sizeof(DecItem) <= 80, "staged item slot");
static_assert(sizeof(ListMeta) <= 32, "staged list metadata slot");

__device__ __forceinline__ DecItem dec_item(const PlanView& pv, int it, int g) {
  DecItem d;
  d.req = pv.item_req[it];
  d.kvh = pv.item_kvh[it];
  const int qt = pv.item_qtile[it];
  d.kb = pv.item_kb[it];
  d.ke = pv.item_ke[it];
  d.slot = pv.item_slot[it];
  d.lq = pv.req_qo_len[d.req];
  d.lk = pv.req_kv_len[d.req];
  d.qo_begin = pv.req_qo_begin[d.req];
  d.page_begin = pv.req_page_begin[d.req];
  d.row0 = qt * pv.T_q;
  d.nrows = min(pv.T_q, d.lq * g - d.row0);
  d.ntiles = (int)((d.ke - d.kb + dec::kTile - 1) / dec::kTile);
  return d;
}

// RoPE of one 16-byte chunk pair in shared memory (R31): 8 elements of the first half (d = i0..i0+7)
// and their partners d + 64 in the second half, rotated by pos * theta_i and rounded back to the
// operand type (the MMA reads them in place).
template <bool kF16>
__device__ __forceinline__ void rope_chunk(uint8_t* lo, uint8_t* hi, int64_t pos, const uint64_t* f, int i0) {
  using T = typename std::conditional<kF16, __half, __nv_bfloat16>::type;
  uint4 a = *reinterpret_cast<uint4*>(lo), b = *reinterpret_cast<uint4*>(hi);
  T* x = reinterpret_cast<T*>(&a);
  T* y = reinterpret_cast<T*>(&b);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float sn, cs;
    rope_sincos(pos, f[i0 + e], sn, cs);
    const float xv = to_f<T>(x[e]), yv = to_f<T>(y[e]);
    x[e] = from_float<T>(xv * cs - yv * sn);
    y[e] = from_float<T>(yv * cs + xv * sn);
  }
  *reinterpret_cast<uint4*>(lo) = a;
  *reinterpret_cast<uint4*>(hi) = b;
}

// Pipeline trace points (BSRA_EXPERIMENTS builds only; scripts/trace_decode.py)
#ifdef BSRA_EXPERIMENTS
#define DEC_TRACE(e) do { if (p.trace) p.trace[(e) * 1024 + blockIdx.x] = (long long)ptx::globaltimer_ns(); } while (0)
// per-tile clock64 events of CTA 0 (index k < 1024): rows 20.. of the trace buffer
#define DEC_TTRACE(e, k) do { if (p.trace && blockIdx.x == 0 && (k) < 1024) p.trace[(20 + (e)) * 1024 + (k)] = clock64(); } while (0)
#else
#define DEC_TRACE(e) do { } while (0)
#define DEC_TTRACE(e, k) do { } while (0)
#endif

// kF16: fp16 q / o (else bf16) at compile time: one code path per instantiation (instruction
// fetch stalls measured on the fp8 kernel when both were inlined). kRope: fused RoPE (R31) —
// eight more warps rotate each landed K tile in shared memory and each item's Q tile before the
// MMA warp reads them (krot / qrot barriers replace full / full_q for S).
// kRow: K/V row gather (tp.cp = 1 cp.async, 2 TMA gather4) instead of per-page TMA boxes — its own
// instantiation, so the box kernel carries none of that code.
// kD: head_dim 128 (two 64-column SW128 halves per row) or 64 (one half: the S MMA takes K = 64,
// the PV MMA keeps M = 128 with O^T rows 64..127 unused and never stored).
// kGrp: K/V tiles group-major — [16 groups of 8 tokens][64-column half][8 rows][128 B] — so ONE TMA
// box of the 5-D pool view (d_lo, token_lo, half, token_hi, page*cs + head) brings a whole page
// (both halves, 4 KB at B_c = 16) where the half-major layout [half][128 rows][128 B] needs one box
// per half: the decode producer is TMA-issue-bound at ~80-90 cycles per small box
// (scripts/tma_issue_bench.cu), so half the boxes per tile. Paged pools only (the 8-token groups
// need page-aligned tiles); the MMA descriptors take SBO = 2048 and the half offset 1024.
template <int kC, int kMask, bool kF16, bool kRope, bool kRow = false, int kD = 128, bool kGrp = false>
__global__ void __launch_bounds__(dec::threads_for(kRope, kRow), 1) tc_decode_kernel(const __grid_constant__ TcParams tp) {
  static_assert(kD == 128 || (kD == 64 && !kRope && !kRow), "head_dim 64: box gather, no RoPE");
  static_assert(!kGrp || (kD == 128 && !kRope && !kRow), "group-major tiles: plain box gather, head_dim 128");
  constexpr int kRowG = kGrp ? 2048 : 1024;                // bytes between 8-row groups of a K/V tile (SBO)
  constexpr int kHalfOff = kGrp ? 1024 : dec::kHalfBytes;  // bytes between the two 64-column halves
  using namespace dec;
  const AttnParams& p = tp.p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* full = bar;                  // [kStages]
  uint64_t* empty = bar + kStages;       // [kStages]
  uint64_t* full_q = bar + 2 * kStages;  // [2]
  uint64_t* empty_q = full_q + 2;        // [2]
  uint64_t* bar_s = empty_q + 2;         // [2] S^T buffer ready
  uint64_t* bar_pv = bar_s + 2;          // [2] PV MMA reading P^T buffer b done
  uint64_t* s_free = bar_pv + 2;         // [2] softmax read S^T buffer b (4 warp arrivals)
  uint64_t* p_full = s_free + 2;         // [2] P^T buffer b written (1 arrival)
  uint64_t* o_free = p_full + 2;         // [2] epilogue read O^T buffer b (1 arrival)
  uint64_t* epi_full = o_free + 2;       // [2] item's row sums / max handed to the epilogue (4 warps)
  uint64_t* epi_empty = epi_full + 2;    // [2] epilogue consumed hand-off buffer b (1 arrival)
  uint64_t* o_full = epi_empty + 2;      // [2] the item's last PV into O^T buffer b completed (commit)
  uint64_t* krot = o_full + 2;           // [kStages] kRope: K tile of the stage rotated
  uint64_t* qrot = krot + kStages;       // [2] kRope: Q buffer rotated
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qrot + 2);
  float* red = reinterpret_cast<float*>(smem + kOffRed);  // [4 warps][kN]
  int* vflags = reinterpret_cast<int*>(red + 4 * kN);     // [2][4] vote flags
  float* hsum = reinterpret_cast<float*>(vflags + 8);      // [2][4 warps][kN] row-sum partials
  float* hmax = hsum + 2 * 4 * kN;                          // [2][kN] running max

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) DEC_TRACE(7);
#ifdef BSRA_EXPERIMENTS
  if (p.trace && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[15 * 1024 + blockIdx.x] = smid + 1;
  }
#endif
  const PlanView pv = load_plan(p.plan);
  const int g = p.g;
  const int it0 = pv.cta_indptr[blockIdx.x], it1 = pv.cta_indptr[blockIdx.x + 1];
  // Every role walks the same queue: its first kStagedItems entries are decoded once here (the
  // plan reads of an item are ~3 dependent global loads, otherwise paid by each role at each item
  // boundary on the critical path)
  DecItem* staged = reinterpret_cast<DecItem*>(smem + kOffItems);
  for (int k = threadIdx.x; k < min(kStagedItems, it1 - it0); k += blockDim.x) staged[k] = dec_item(pv, it0 + k, g);
  auto item_at = [&](int it) { return it - it0 < kStagedItems ? staged[it - it0] : dec_item(pv, it, g); };

  // producer warps: warp 0 (Q and K), 10 (V); gather4: warps 0, 10..16 (quarter x half of the rows)
#ifndef BSRA_BOX_PRODUCERS
#define BSRA_BOX_PRODUCERS 2
#endif
  const int nprod = kRope ? BSRA_ROPE_PRODUCERS
                          : (kRow && tp.cp == 1) ? 1 : (kRow && tp.cp == 2 ? 8 : BSRA_BOX_PRODUCERS);
  if (threadIdx.x == 0) {
    DEC_TRACE(0);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], kRow && tp.cp == 1 ? 32 : nprod);  // cp.async gather: one arrival per lane
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&krot[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&full_q[b], 1);
      ptx::mbar_init(&empty_q[b], 1);
      ptx::mbar_init(&bar_s[b], 1);
      ptx::mbar_init(&bar_pv[b], 1);
      ptx::mbar_init(&s_free[b], 4);
      ptx::mbar_init(&p_full[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&o_free[b], 1);
      ptx::mbar_init(&epi_full[b], 4);
      ptx::mbar_init(&epi_empty[b], 1);
      ptx::mbar_init(&o_full[b], 1);
      ptx::mbar_init(&qrot[b], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp >= 1 && warp <= 4) {  // zero both P^T buffers once: rows >= kC stay zero for the kernel's lifetime
    uint4* pz = reinterpret_cast<uint4*>(smem + kOffP);
    for (int i = threadIdx.x - 32; i < 2 * kPBytes / 16; i += 128) pz[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async();
  }
  if (warp == 5) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) DEC_TRACE(6);
  pdl_launch_dependents();  // PDL: the next kernel's CTAs may take SMs this grid releases
  // debug (p.trace set): per-CTA start / end time, globaltimer ns (scripts/cta_balance.py)
#ifdef BSRA_EXPERIMENTS
  if (p.trace && threadIdx.x == 0) p.trace[16 * 1024 + blockIdx.x] = (long long)ptx::globaltimer_ns();
#endif

  // producer role: warp 0, then warps 10.. (plain / row variants) or warp 18 (RoPE variant)
  const int prole = warp == 0 ? 0 : (!kRope && warp >= 10 ? warp - 9 : (kRope && warp == 18 ? 1 : -1));
  if (prole >= 0) {
    // ============================ TMA producers ============================
    // role 0: Q + K (box path) / K half 0 (gather4) / everything (cp.async, RoPE variant); role 1:
    // V / K half 1; roles 2, 3: V halves 0 / 1 (gather4). Every role walks the same tile sequence.
    if (prole < nprod) {
      if (lane == 0) {
        if (prole == 0) ptx::tma_prefetch_desc(&tp.tq);
        ptx::tma_prefetch_desc(&tp.tk);
        ptx::tma_prefetch_desc(&tp.tv);
      }
      const int B = tp.box_tok;
      int stage = 0;
      int tcount = 0;  // trace index
      uint32_t ephase = 1;  // fresh barriers: waiting on parity 1 passes
      uint32_t qphase[2] = {1, 1};
      int qb = 0;
      if (lane == 0) DEC_TRACE(11);
      for (int it = it0; it < it1; ++it) {
        const DecItem d = item_at(it);
        // ---- Q tile: 16 fused rows = q_tb tokens x q_hb heads, two 64-column halves
        if (lane == 0 && prole == 0) {
          ptx::mbar_wait(&empty_q[qb], qphase[qb]);
          ptx::mbar_arrive_expect_tx(&full_q[qb], kD == 128 ? kQBytes : kQBytes / 2);
          const int head0 = d.kvh * g + (g > kN ? d.row0 % g : 0);
          const int tok0 = (int)d.qo_begin + d.row0 / g;
          uint8_t* qdst = smem + kOffQ + qb * kQBytes;
          ptx::tma_load_3d(qdst, &tp.tq, &full_q[qb], 0, head0, tok0);
          if (kD == 128) ptx::tma_load_3d(qdst + kN * 128, &tp.tq, &full_q[qb], 64, head0, tok0);
        }
        qphase[qb] ^= 1;
        qb ^= 1;
        // ---- K/V tiles
        for (int ti = 0; ti < d.ntiles; ++ti) {
          const int64_t t0 = d.kb + (int64_t)ti * kTile;
          if (kRow && tp.cp == 2) {
            // TMA gather4 (sm_100): the K/V pools as 2-D [rows, D] tensors (a (page, slot, head) row
            // is D contiguous elements); lane l loads token rows 4l .. 4l+3 of the tile, both
            // 64-column halves of K and V: 4 instructions per lane, 128 per 64 KB tile, any page
            // size. Rows past the chunk repeat its last row (masked in S, zeroed in V).
            int rows[4];
  #pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int64_t t = imin64(t0 + 4 * lane + j, d.ke - 1);
              const int64_t pg = __ldg(p.page_indices + d.page_begin + t / p.page_size);
              rows[j] = (int)(pg * tp.row_s0 + (t % p.page_size) * tp.row_s1 + d.kvh * tp.row_s2);
            }
            if (lane == 0) {
              ptx::mbar_wait(&empty[stage], ephase);
              ptx::mbar_arrive_expect_tx(&full[stage], (uint32_t)kStageBytes / 8);
            }
            __syncwarp();
            // role r: quarter q = r & 3 (K or V = q >> 1, column half = q & 1), lanes 16 (r >> 2) .. +15
            const int q = prole & 3;
            if ((lane >> 4) == (prole >> 2)) {
              uint8_t* dst = smem + stage * kStageBytes + lane * 4 * 128 + (q >> 1) * kKVBytes + (q & 1) * kHalfBytes;
              ptx::tma_gather4(dst, (q >> 1) ? &tp.tv : &tp.tk, &full[stage], (q & 1) * 64, rows[0], rows[1], rows[2],
                               rows[3]);
            }
            __syncwarp();
          } else if (kRow) {
            // 16-byte cp.async gather, any page size (small pages, B_c not dividing 128): per
            // instruction the warp moves 4 token rows x 128 B (lane = chunk c of row sub), written
            // at the SW128 position TMA would use; rows past the chunk are zero-filled (no read).
            const int c8 = lane & 7, sub = lane >> 3;
            ptx::mbar_wait(&empty[stage], ephase);
            const uint32_t sK = ptx::smem_u32(smem + stage * kStageBytes), sV = sK + kKVBytes;
            const uint16_t* kg = reinterpret_cast<const uint16_t*>(p.k);
            const uint16_t* vg = reinterpret_cast<const uint16_t*>(p.v);
  #pragma unroll 1
            for (int rb0 = 0; rb0 < kTile / 4; rb0 += 8) {
              int64_t ko[8], vo[8];
              bool ok[8];
  #pragma unroll
              for (int u = 0; u < 8; ++u) {  // the 8 rows' page ids first (independent loads)
                const int64_t t = t0 + 4 * (rb0 + u) + sub;
                ok[u] = t < d.ke;
                int64_t pg = 0, sl;
                if (p.kv_ragged) {
                  sl = d.page_begin + t;
                } else {
                  pg = ok[u] ? __ldg(p.page_indices + d.page_begin + t / p.page_size) : 0;
                  sl = t % p.page_size;
                }
                ko[u] = ok[u] ? pg * p.ks0 + sl * p.ks1 + (int64_t)d.kvh * p.ks2 + c8 * 8 : 0;
                vo[u] = ok[u] ? pg * p.vs0 + sl * p.vs1 + (int64_t)d.kvh * p.vs2 + c8 * 8 : 0;
              }
  #pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int r = 4 * (rb0 + u) + sub;
                const uint32_t sw = (uint32_t)(r * 128 + ((c8 ^ (r & 7)) << 4));
                cp_async16_zfill(sK + sw, kg + ko[u], ok[u]);
                cp_async16_zfill(sK + kHalfBytes + sw, kg + ko[u] + 64, ok[u]);
                cp_async16_zfill(sV + sw, vg + vo[u], ok[u]);
                cp_async16_zfill(sV + kHalfBytes + sw, vg + vo[u] + 64, ok[u]);
              }
            }
            cp_async_mbar_arrive_noinc(&full[stage]);
          } else {
            // TMA: lane j handles sub-block j (one page, or 128 tokens of a big page)
            const int n = (int)imin64(kTile, d.ke - t0);
            const int nsub = (n + B - 1) / B;
            int page = 0, off = 0;
            if (lane < nsub) {
              const int64_t tok = t0 + (int64_t)lane * B;
              if (p.kv_ragged) {  // contiguous KV: token coordinate, no page table
                off = (int)(d.page_begin + tok);
              } else {
                page = __ldg(p.page_indices + d.page_begin + tok / p.page_size);
                off = (int)(tok % p.page_size);
              }
            }
            // role 0 loads K, role 1 V (a single role in the RoPE variant: both)
            if (lane == 0) {
              ptx::mbar_wait(&empty[stage], ephase);
              if (prole == 0) DEC_TTRACE(0, tcount);
              ptx::mbar_arrive_expect_tx(&full[stage], (uint32_t)nsub * B * (kD * 4) / nprod);
            }
            __syncwarp();
            if (lane == 0 && it == it0 && ti == 0 && prole == 0) DEC_TRACE(8);
            const bool doK = prole == 0, doV = prole == 1 || nprod == 1;
            if (kGrp && lane < nsub) {  // one box per page: 8-token groups [lane*B/8, (lane+1)*B/8) of the tile
              uint8_t* kd = smem + stage * kStageBytes + (lane * B >> 3) * 2048;
              uint8_t* vd = kd + kKVBytes;
              const int c4 = page * tp.cs + d.kvh;
              if (doK) ptx::tma_load_5d(kd, &tp.tk, &full[stage], 0, 0, 0, off >> 3, c4);
              if (doV) ptx::tma_load_5d(vd, &tp.tv, &full[stage], 0, 0, 0, off >> 3, c4);
            } else if (lane < nsub) {
              uint8_t* kd = smem + stage * kStageBytes + lane * B * 128;
              uint8_t* vd = kd + kKVBytes;
              if (doK) {
                ptx::tma_load_4d(kd, &tp.tk, &full[stage], 0, d.kvh, off, page);
                if (kD == 128) ptx::tma_load_4d(kd + kHalfBytes, &tp.tk, &full[stage], 64, d.kvh, off, page);
              }
              if (doV) {
                ptx::tma_load_4d(vd, &tp.tv, &full[stage], 0, d.kvh, off, page);
                if (kD == 128) ptx::tma_load_4d(vd + kHalfBytes, &tp.tv, &full[stage], 64, d.kvh, off, page);
              }
            }
            __syncwarp();
          }
          ++tcount;
          if (++stage == kStages) {
            stage = 0;
            ephase ^= 1;
          }
        }
      }
    }  // prole < nprod
  } else if (warp == 5) {
    // ================================ MMA issuer ================================
    // One flat stream of tiles across the CTA's items: S(k) as soon as K(k) landed and the softmax
    // has read the S^T buffer, then PV(k-1) once P(k-1) is written. At an item boundary the next
    // item's first S is issued BEFORE the previous item's last PV, so the softmax warps go on to
    // the next item while that PV runs (the epilogue waits for it through o_full).
    const uint32_t fmt = kF16 ? 0u : 1u;
    const uint32_t idS = ptx::idesc_f16(fmt, 128, kN, 0, 0);  // A = K (K-major), B = Q (K-major)
    const uint32_t idO = ptx::idesc_f16(fmt, 128, kN, 1, 0);  // A = V^T (MN-major), B = P^T (K-major)
    const uint32_t sbase = ptx::smem_u32(smem);
    int stage = 0, sb = 0, pb = 0, qb = 0, ob = 0;
    int tcount = 0;
    uint32_t fphase = 0;
    uint32_t ofph[2] = {1, 1};
    uint32_t sfph[2] = {1, 1}, pfph[2] = {0, 0}, qphase[2] = {0, 0};
    struct PendingPV {
      int st, ti, ob;
      bool last, valid;
    } pend = {0, 0, 0, false, false};
    auto issue_pv = [&](const PendingPV& x) {  // PV of tile x.ti of an item, staged in ring stage x.st
      ptx::mbar_wait(&p_full[pb], pfph[pb]);
      pfph[pb] ^= 1;
      if (x.ti == 0) {  // the item's first PV overwrites O[ob]: the epilogue two items back read it
        ptx::mbar_wait(&o_free[x.ob], ofph[x.ob]);
        ofph[x.ob] ^= 1;
      }
      ptx::tc_fence_after();
      const uint64_t a0 = ptx::smem_desc_sw128(sbase + x.st * kStageBytes + kKVBytes, kHalfOff, kRowG);
      const uint64_t b0 = ptx::smem_desc_sw128(sbase + kOffP + pb * kPBytes, 16, 1024);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t sbo = (uint64_t)((kk >> 2) * (kN * 128 >> 4) + (kk & 3) * 2);
        ptx::mma_f16_ss_warp(tmem + 32 + x.ob * 16, a0 + (uint64_t)(kk * (2 * kRowG >> 4)), b0 + sbo, idO,
                             (x.ti > 0 || kk > 0) ? 1u : 0u);
      }
      ptx::mma_commit_warp(&empty[x.st]);  // K/V stage free once these MMAs complete
      ptx::mma_commit_warp(&bar_pv[pb]);
      if (x.last) ptx::mma_commit_warp(&o_full[x.ob]);  // O[ob] final: the epilogue may read it
      pb ^= 1;
    };
    for (int it = it0; it < it1; ++it) {
      const DecItem d = item_at(it);
      ptx::mbar_wait(kRope ? &qrot[qb] : &full_q[qb], qphase[qb]);
      qphase[qb] ^= 1;
      if (lane == 0 && it == it0) DEC_TRACE(9);
      if (d.ntiles == 0) {
        ptx::mbar_arrive_warp(&empty_q[qb]);
        qb ^= 1;
        continue;
      }
      const uint64_t bq = ptx::smem_desc_sw128(sbase + kOffQ + qb * kQBytes, 16, 1024);
      for (int ti = 0; ti < d.ntiles; ++ti) {
        ptx::mbar_wait(kRope ? &krot[stage] : &full[stage], fphase);
        if (lane == 0 && it == it0 && ti == 0) DEC_TRACE(10);
        if (lane == 0) DEC_TTRACE(1, tcount);
        ptx::mbar_wait(&s_free[sb], sfph[sb]);
        sfph[sb] ^= 1;
        if (lane == 0) DEC_TTRACE(2, tcount);
        ++tcount;
        if (kRow && tp.cp == 1) ptx::fence_proxy_async();  // cp.async (generic-proxy) writes -> tensor core
        ptx::tc_fence_after();
        const uint64_t a0 = ptx::smem_desc_sw128(sbase + stage * kStageBytes, 16, kRowG);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t sa = (uint64_t)((kk >> 2) * (kHalfOff >> 4) + (kk & 3) * 2);
          const uint64_t sbo = (uint64_t)((kk >> 2) * (kN * 128 >> 4) + (kk & 3) * 2);
          ptx::mma_f16_ss_warp(tmem + sb * 16, a0 + sa, bq + sbo, idS, kk > 0);
        }
        ptx::mma_commit_warp(&bar_s[sb]);
        if (ti + 1 == d.ntiles) ptx::mma_commit_warp(&empty_q[qb]);  // last reader of this Q buffer
        sb ^= 1;
        if (pend.valid) issue_pv(pend);
        pend = {stage, ti, ob, ti + 1 == d.ntiles, true};
        if (++stage == kStages) {
          stage = 0;
          fphase ^= 1;
        }
      }
      qb ^= 1;
      ob ^= 1;
    }
    if (pend.valid) issue_pv(pend);
  } else if (warp <= 4) {
    // ============================ softmax warps (1..4) ============================
    const int ct = threadIdx.x - 32;         // 0..127
    const int q4 = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = q4 * 32 + lane;          // TMEM lane: token (softmax) / head-dim d (output)
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    int ob = 0;                              // O^T buffer of the current item (32 / 48)
    uint32_t eeph[2] = {1, 1};               // epi_empty parities (fresh: first waits pass)
    // pipeline state (identical in every softmax thread)
    int stage = 0;            // ring stage of the tile being processed
    uint32_t fphase = 0;      // its full-barrier parity
    uint32_t sph[2] = {0, 0}, pvph[2] = {0, 0};
    bool pv_pending[2] = {false, false};
    int sbuf = 0;             // S^T buffer of the tile being processed
    int pbuf = 0;             // P^T buffer to write next
    int tpar = 0;             // tile count (parity selects the vote-flag buffer)
    auto wait_pv = [&](int b) {
      if (pv_pending[b]) {
        ptx::mbar_wait(&bar_pv[b], pvph[b]);
        pvph[b] ^= 1;
        pv_pending[b] = false;
      }
    };

    for (int it = it0; it < it1; ++it) {
      const DecItem d = item_at(it);
      if (d.ntiles == 0) continue;  // empty item: the epilogue warps write the empty state
      const uint32_t tO = tmem + lane_addr + 32 + ob * 16;
      float m[kC], lp[kC], aslope[kC];
      int64_t lim[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        m[c] = -INFINITY;
        lp[c] = 0.f;
        const int tok = (d.row0 + c) / g;
        aslope[c] = p.alibi ? alibi_slope_raw(p, d.kvh * g + (d.row0 + c) % g) : 0.f;  // ALiBi (R30)
        lim[c] = kMask == 1 ? d.lk - d.lq + tok : (kMask == 2 ? p.mask_indptr[d.req] + (int64_t)tok * d.lk : 0);
      }
      for (int ti = 0; ti < d.ntiles; ++ti) {
        const int64_t t0 = d.kb + (int64_t)ti * kTile;
        const int n = (int)imin64(kTile, d.ke - t0);
        ptx::mbar_wait(&bar_s[sbuf], sph[sbuf]);
        sph[sbuf] ^= 1;
        if (ct == 0 && it == it0 && ti == 0) DEC_TRACE(1);
        if (ct == 0) DEC_TTRACE(3, tpar);
        ptx::tc_fence_after();
        float s[kC];
        ptx::tmem_ld<kC>(tmem + lane_addr + sbuf * 16, s);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&s_free[sbuf]);  // the MMA warp may reuse this S^T buffer
        // rows past the chunk: zero V so 0 * garbage cannot poison O (the cp.async gather already
        // zero-filled them)
        if (n < kTile && row >= n && !(kRow && tp.cp == 1)) {
          ptx::mbar_wait(&full[stage], fphase);  // (already complete) orders the TMA writes before ours
          uint8_t* vS = smem + stage * kStageBytes + kKVBytes;
          uint4 z = make_uint4(0, 0, 0, 0);
          const int roff = kGrp ? (row >> 3) * 2048 + (row & 7) * 128 : row * 128;
          uint4* v0 = reinterpret_cast<uint4*>(vS + roff);
          uint4* v1 = reinterpret_cast<uint4*>(vS + kHalfOff + roff);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v0[j] = z;
            v1[j] = z;
          }
        }
        // ---- mask + scale
        const int64_t t = t0 + row;
        const bool tok_ok = row < n;
#pragma unroll
        for (int c = 0; c < kC; ++c) {
          bool vis = tok_ok && c < d.nrows;
          if (kMask == 1) vis = vis && t <= lim[c];
          if (kMask == 2) vis = vis && mask_bit(p.mask, lim[c] + t);
          if (p.window > 0) vis = vis && t >= d.lk - d.lq + (d.row0 + c) / g - p.window + 1;  // R26
          float sc = p.soft_cap > 0.f ? soft_cap_raw(p, s[c]) : s[c];                      // R27
          if (p.alibi) sc += aslope[c] * (float)(t - (d.lk - d.lq + (d.row0 + c) / g));  // R30
          s[c] = vis ? sc * p.scale_log2 : -INFINITY;
        }
        // ---- stale-max softmax (lazy rescale, exact: o and lse use the same max): P = 2^(s - m)
        // with the running max m; only when some score exceeds m by more than 2^8 (every item's
        // first tile) do the warps reduce the tile max, rescale O and recompute P. The common
        // path has no shuffles and one barrier: a warp vote and a per-warp flag (double-buffered
        // by tile parity) read after it.
        // An item's first tile always takes the reduction (the running max is -inf), so it skips
        // the vote and the speculative exp / P store / barrier of the common path.
        const bool first = ti == 0;
        int* flags = vflags + (tpar & 1) * 4;
        float pr[kC];
        if (!first) {
          bool over = false;
#pragma unroll
          for (int c = 0; c < kC; ++c) over |= s[c] > m[c] + kRescaleThresh;
          over = __any_sync(0xffffffffu, over);
          if (lane == 0) flags[q4] = over ? 1 : 0;
#pragma unroll
          for (int c = 0; c < kC; ++c) pr[c] = s[c] == -INFINITY ? 0.f : exp2f(s[c] - m[c]);
        }
        wait_pv(pbuf);  // the PV MMA that read this P^T buffer two tiles ago is done
        // ---- P^T (K-major, SW128): row c, token `row`
        uint8_t* pa = smem + kOffP + pbuf * kPBytes + (row >> 6) * (kN * 128);
        const int tt = row & 63;
        auto store_p = [&]() {
#pragma unroll
          for (int c = 0; c < kC; ++c) {
            const uint32_t off = (c >> 3) * 1024 + (c & 7) * 128 + ((((tt >> 3) ^ (c & 7)) << 4) | ((tt & 7) << 1));
            if constexpr (kF16) *reinterpret_cast<__half*>(pa + off) = __float2half_rn(pr[c]);
            else *reinterpret_cast<__nv_bfloat16*>(pa + off) = __float2bfloat16_rn(pr[c]);
          }
        };
        if (!first) {
          store_p();
          ptx::fence_proxy_async();  // P (and zeroed V rows) visible to the tensor core
          ptx::named_bar_sync(1, 128);
        }
        if (first || (flags[0] | flags[1] | flags[2] | flags[3])) {  // slow path
          float mx[kC];
#pragma unroll
          for (int c = 0; c < kC; ++c) mx[c] = s[c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int c = 0; c < kC; ++c) mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
          }
          if (lane == 0) {
#pragma unroll
            for (int c = 0; c < kC; ++c) red[q4 * kN + c] = mx[c];
          }
          ptx::named_bar_sync(1, 128);
          float alpha[kC];
          bool rescale = false;
#pragma unroll
          for (int c = 0; c < kC; ++c) {
            const float mt = fmaxf(fmaxf(red[c], red[kN + c]), fmaxf(red[2 * kN + c], red[3 * kN + c]));
            alpha[c] = 1.f;
            if (mt > m[c] + kRescaleThresh) {
              if (m[c] != -INFINITY) {
                alpha[c] = exp2f(m[c] - mt);
                rescale = true;
              }
              m[c] = mt;
            }
            pr[c] = s[c] == -INFINITY ? 0.f : exp2f(s[c] - m[c]);
            lp[c] *= alpha[c];
          }
          if (rescale) {  // bring O^T to the new max (PV(t-1) done; PV(t) waits for p_full)
            wait_pv(pbuf ^ 1);
            ptx::tc_fence_after();
            float ov[kC];
            ptx::tmem_ld<kC>(tO, ov);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < kC; ++c) ov[c] *= alpha[c];
            ptx::tmem_st<kC>(tO, ov);
            ptx::tmem_st_wait();
          }
          store_p();
          ptx::fence_proxy_async();
          ptx::tc_fence_before();
          ptx::named_bar_sync(1, 128);
        }
#pragma unroll
        for (int c = 0; c < kC; ++c) lp[c] += pr[c];
        if (ct == 0) ptx::mbar_arrive(&p_full[pbuf]);  // the MMA warp issues PV(t)
        if (ct == 0) DEC_TTRACE(4, tpar);
        ++tpar;
        pv_pending[pbuf] = true;
        pbuf ^= 1;
        sbuf ^= 1;
        if (++stage == kStages) {
          stage = 0;
          fphase ^= 1;
        }
      }
      // ---- hand the item to the epilogue warps: per-warp row-sum partials and the running max (the
      // item's last PV may still run: the epilogue waits for it on o_full, so the softmax warps go on)
      float x[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        x[c] = lp[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x[c] += __shfl_xor_sync(0xffffffffu, x[c], o);
      }
      ptx::mbar_wait(&epi_empty[ob], eeph[ob]);
      eeph[ob] ^= 1;
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < kC; ++c) hsum[(ob * 4 + q4) * kN + c] = x[c];
        if (q4 == 0) {
#pragma unroll
          for (int c = 0; c < kC; ++c) hmax[ob * kN + c] = m[c];
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&epi_full[ob]);
      ob ^= 1;
    }
    if (ct == 0) DEC_TRACE(2);
  } else if (kRope && warp >= 10) {
    // ====== RoPE warps (10..17): rotate Q (per item) and K (per tile) in shared memory (R31) ======
    const int rt = threadIdx.x - dec::kThreads;  // 0..255
    int stage = 0, qb = 0;
    uint32_t fphase = 0, qph[2] = {0, 0};
    const uint64_t* f = p.rope_f;
    const int ri = rt & 63, rgrp = rt >> 6;  // K: pair index and row group (rows = rgrp mod 4)
    float s2, c2;
    rope_sincos_precise(4, f[ri], s2, c2);  // the per-step rotation by 4 theta_i (1 ulp)
    for (int it = it0; it < it1; ++it) {
      const DecItem d = item_at(it);
      ptx::mbar_wait(&full_q[qb], qph[qb]);
      qph[qb] ^= 1;
      {  // Q: 16 rows x 8 chunk pairs; fused row c is token (row0 + c) / g at l_kv - l_qo + token
        const int c = rt >> 3, ch = rt & 7;
        if (d.ntiles > 0 && rt < 128 && c < kC && c < d.nrows) {
          uint8_t* q0 = smem + kOffQ + qb * kQBytes + c * 128 + ((ch ^ (c & 7)) << 4);
          rope_chunk<kF16>(q0, q0 + kN * 128, d.lk - d.lq + (d.row0 + c) / g, f, ch * 8);
        }
        ptx::fence_proxy_async();  // generic-proxy writes visible to the tensor core
        ptx::named_bar_sync(3, 256);
        if (rt == 0) ptx::mbar_arrive(&qrot[qb]);
      }
      qb ^= 1;
      for (int ti = 0; ti < d.ntiles; ++ti) {
        ptx::mbar_wait(&full[stage], fphase);
        // K: thread = (pair i, row group); it walks rows grp, grp + 4, ... of the tile, so the
        // angle (t0 + r) theta_i advances by the constant 4 theta_i: one sincos per tile and a
        // rotation recurrence per row (fp32, 32 steps: ~1e-6 relative drift, far below the bf16
        // rounding of the rotated key). Lanes = consecutive pairs: 2-byte accesses to one row's
        // 64-byte run, conflict-free.
        const int64_t t0 = d.kb + (int64_t)ti * kTile;
        float cs, sn;
        rope_sincos(t0 + rgrp, f[ri], sn, cs);
        uint8_t* kst = smem + stage * kStageBytes;
        const int cofs = (ri & 7) << 1;  // byte offset of element ri inside its 16-byte chunk
        using T = typename std::conditional<kF16, __half, __nv_bfloat16>::type;
#pragma unroll 1
        for (int r0 = rgrp; r0 < kTile; r0 += 32) {  // 8 rows per batch: loads, math, stores
          T xv[8], yv[8];                             // (explicit batches: a store does not block
#pragma unroll                                        //  the next rows' loads on may-alias)
          for (int u = 0; u < 8; ++u) {
            const int r = r0 + 4 * u;
            const int off = r * 128 + (((ri >> 3) ^ (r & 7)) << 4) + cofs;
            xv[u] = *reinterpret_cast<const T*>(kst + off);
            yv[u] = *reinterpret_cast<const T*>(kst + kHalfBytes + off);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float x = to_f<T>(xv[u]), y = to_f<T>(yv[u]);
            xv[u] = from_float<T>(x * cs - y * sn);
            yv[u] = from_float<T>(y * cs + x * sn);
            const float c1 = cs * c2 - sn * s2;  // angle += 4 theta_i
            sn = sn * c2 + cs * s2;
            cs = c1;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = r0 + 4 * u;
            const int off = r * 128 + (((ri >> 3) ^ (r & 7)) << 4) + cofs;
            *reinterpret_cast<T*>(kst + off) = xv[u];
            *reinterpret_cast<T*>(kst + kHalfBytes + off) = yv[u];
          }
        }
        ptx::fence_proxy_async();
        ptx::named_bar_sync(3, 256);
        if (rt == 0) ptx::mbar_arrive(&krot[stage]);
        if (++stage == kStages) {
          stage = 0;
          fphase ^= 1;
        }
      }
    }
  } else if (warp >= 6) {
    // ====== epilogue warps (6..9): thread = TMEM lane = head-dim row d of O^T; normalise, write ======
    const int et = threadIdx.x - 192;        // 0..127
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    int ob = 0;
    uint32_t efph[2] = {0, 0};
    // merge-list metadata of the staged split items, resolved while the first tiles stream in
    ListMeta* smeta = reinterpret_cast<ListMeta*>(smem + kOffMeta);
    const int nstaged = min(kStagedItems, it1 - it0);
    if (p.fused_merge) {
      for (int k = et; k < nstaged; k += 128)
        if (staged[k].slot >= 0) smeta[k] = list_meta(pv, list_of_slot(pv, staged[k].slot), g);
      ptx::named_bar_sync(2, 128);
    }
    pdl_wait();  // PDL: the previous kernel on the stream has completed before we write
    if (et == 0) DEC_TRACE(3);
    for (int it = it0; it < it1; ++it) {
      const DecItem d = item_at(it);
      float ov[kC], l[kC], mm[kC];
      if (d.ntiles > 0) {
        ptx::mbar_wait(&epi_full[ob], efph[ob]);
        ptx::mbar_wait(&o_full[ob], efph[ob]);  // the item's last PV completed
        efph[ob] ^= 1;
        if (et == 0) DEC_TTRACE(5, it - it0);
        ptx::tc_fence_after();
        ptx::tmem_ld<kC>(tmem + lane_addr + 32 + ob * 16, ov);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < kC; ++c) {
          const float* hs = hsum + ob * 4 * kN + c;
          l[c] = (hs[0] + hs[kN]) + (hs[2 * kN] + hs[3 * kN]);
          mm[c] = hmax[ob * kN + c];
        }
        ptx::tc_fence_before();
        ptx::named_bar_sync(2, 128);  // all lanes of O[ob] and the hand-off buffer read
        if (et == 0) {
          ptx::mbar_arrive(&o_free[ob]);     // the item two ahead may overwrite O[ob]
          ptx::mbar_arrive(&epi_empty[ob]);  // and the softmax may refill the hand-off buffer
        }
        ob ^= 1;
      } else {
#pragma unroll
        for (int c = 0; c < kC; ++c) {
          ov[c] = 0.f;
          l[c] = 0.f;
          mm[c] = -INFINITY;
        }
      }
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        if (c < d.nrows && row < kD) {
          const bool empty_row = !(l[c] > 0.f);
          const float val = empty_row ? 0.f : ov[c] / l[c];
          const float lse = empty_row ? -INFINITY : (mm[c] + __log2f(l[c])) * kLn2;
          const int f = d.row0 + c;
          const int tok = f / g, head = d.kvh * g + f % g;
          if (d.slot < 0) {
            const int64_t orow = (d.qo_begin + tok) * p.H_qo + head;
            if (p.o_f32) reinterpret_cast<float*>(p.o)[orow * kD + row] = val;
            else if constexpr (kF16) reinterpret_cast<__half*>(p.o)[orow * kD + row] = __float2half_rn(val);
            else reinterpret_cast<__nv_bfloat16*>(p.o)[orow * kD + row] = __float2bfloat16_rn(val);
            if (p.lse && row == 0) p.lse[orow] = lse;
          } else {
            const int64_t prow = (int64_t)d.slot * p.T_slot + c;
            p.part_o[prow * kD + row] = val;
            if (row == 0) p.part_lse[prow] = lse;
          }
        }
      }
      if (et == 0 && it + 1 == it1) DEC_TRACE(4);
      if (et == 0) DEC_TTRACE(6, it - it0);
      if (d.slot >= 0 && p.fused_merge) {  // split item: the CTA completing its merge list folds it
        volatile int* s_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
        const ListMeta* pre = it - it0 < kStagedItems ? smeta + (it - it0) : nullptr;
        if constexpr (kF16) fused_contraction_meta<__half, kD>(p, pv, pre, d.slot, et, 128, 2, s_flag);
        else fused_contraction_meta<__nv_bfloat16, kD>(p, pv, pre, d.slot, et, 128, 2, s_flag);
      }
    }
    if (et == 0) DEC_TRACE(5);
  }
  ptx::tc_fence_before();
  __syncthreads();
#ifdef BSRA_EXPERIMENTS
  if (p.trace && threadIdx.x == 0) p.trace[17 * 1024 + blockIdx.x] = (long long)ptx::globaltimer_ns();
#endif
  if (warp == 5) ptx::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace bsra
