// merge.cuh — the attention-state operator ⊕ (§2.2) on the GPU.
//
//  * fused_contraction: the plan-driven "contraction" stage, fused into the persistent
//    attention kernels: for every merge list (one per split (request, kv head, q tile))
//    fold ⊕ over its partial slots in the plan's fixed order (ascending kv_begin, R17)
//    — a left fold, no atomics on values (an arrival counter only elects the merging CTA),
//    so results are deterministic.
//  * merge_states_kernel / merge_many_kernel: ⊕ of whole state tensors (composable formats,
//    P:172-174; cross-GPU sequence split).
// One warp per state; each lane owns D/32 consecutive dims. Max-shifted form; the empty state
// (o = 0, lse = -inf) is the identity (R3).
#pragma once
#include "common.cuh"

namespace bsra {

// acc <- acc ⊕ (o, l), fp32, lane-local dims
template <int kPer>
__device__ __forceinline__ void oplus(float* acc, float& acc_lse, const float* o, float l) {
  const float mx = fmaxf(acc_lse, l);
  if (mx == -INFINITY) return;  // both empty
  const float wa = __expf(acc_lse - mx), wb = __expf(l - mx);
  const float inv = 1.f / (wa + wb);
#pragma unroll
  for (int j = 0; j < kPer; ++j) acc[j] = (wa * acc[j] + wb * o[j]) * inv;
  acc_lse = mx + __logf(wa + wb);
}

template <typename TO, int D>
__device__ __forceinline__ void store_row(void* out, int64_t row, int lane, const float* acc, int o_f32) {
  constexpr int kPer = D / 32;
  if (o_f32) {
    float* o = reinterpret_cast<float*>(out) + row * D + lane * kPer;
#pragma unroll
    for (int j = 0; j < kPer; ++j) o[j] = acc[j];
  } else {
    TO* o = reinterpret_cast<TO*>(out) + row * D + lane * kPer;
#pragma unroll
    for (int j = 0; j < kPer; ++j) o[j] = from_float<TO>(acc[j]);
  }
}

// ---------------------------------------------------------------------------------------------
// Fused contraction ("We merge the two stages into one persistent kernel"): after the
// `nthr` threads of a CTA (or warpgroup) have written the partial rows of a split item, they
// call this. The CTA whose arrival completes a merge list folds that list's slots in the plan's
// fixed order (deterministic: the result does not depend on which CTA merges) and resets the
// list's counter for the next launch. Partials of other CTAs are read with ld.global.cg (L1 is
// not coherent across SMs).
__device__ __forceinline__ int list_of_slot(const PlanView& pv, int slot) {
  int lo = 0, hi = pv.n_lists;  // list_indptr[lo] <= slot < list_indptr[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pv.list_indptr[mid] <= slot) lo = mid;
    else hi = mid;
  }
  return lo;
}

// A merge list's metadata (everything the merging CTA needs besides the partials). The decode
// kernels resolve it for their staged items while the K/V stream runs, so the tail of a launch
// does not pay the slot -> list binary search and the plan reads (dependent global loads) after
// the arrival.
struct ListMeta {
  int l, s0, s1, kvh, qt, nrows;
  int64_t qo_begin;
};

__device__ __forceinline__ ListMeta list_meta(const PlanView& pv, int l, int g) {
  ListMeta m;
  m.l = l;
  m.s0 = pv.list_indptr[l];
  m.s1 = pv.list_indptr[l + 1];
  const int req = pv.list_req[l];
  m.kvh = pv.list_kvh[l];
  m.qt = pv.list_qtile[l];
  m.nrows = min(pv.T_q, pv.req_qo_len[req] * g - m.qt * pv.T_q);
  m.qo_begin = pv.req_qo_begin[req];
  return m;
}

template <typename TO, int D>
__device__ __forceinline__ void fused_contraction_meta(const AttnParams& p, const PlanView& pv, const ListMeta* pre,
                                                       int slot, int tid, int nthr, int bar_id, volatile int* s_flag) {
  __threadfence();  // this thread's partial writes are visible device-wide
  asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nthr) : "memory");
  if (tid == 0) {
    const int l = pre ? pre->l : list_of_slot(pv, slot);
    const int len = pre ? pre->s1 - pre->s0 : pv.list_indptr[l + 1] - pv.list_indptr[l];
    const int old = atomicAdd(p.counters + l, 1);
    const bool last = old == len - 1;
    if (last) p.counters[l] = 0;  // every other arrival of this launch has happened
    *s_flag = last ? l : -1;
  }
  asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nthr) : "memory");
  const int l = *s_flag;
  if (l >= 0) {
    __threadfence();  // acquire: the other CTAs' partials are visible
    const ListMeta lm = pre ? *pre : list_meta(pv, l, p.g);
    const int kvh = lm.kvh, qt = lm.qt, nrows = lm.nrows, s0 = lm.s0, s1 = lm.s1;
    // ⊕ over the list in closed form (max-shifted): per row one warp forms the slot weights
    // w_s = e^{lse_s - m} once, then lanes accumulate D/32 contiguous dims per slot in slot order.
    constexpr int kPer = D / 32;
    const int lane = tid & 31, nwarps = nthr >> 5;
    for (int r = tid >> 5; r < nrows; r += nwarps) {
      float m = -INFINITY;
      for (int s = s0 + lane; s < s1; s += 32)
        m = fmaxf(m, __ldcg(p.part_lse + (int64_t)pv.list_slot[s] * p.T_slot + r));
      m = warp_max(m);
      float acc[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) acc[j] = 0.f;
      float tot = 0.f;
      if (m != -INFINITY) {
        for (int sb = s0; sb < s1; sb += 8) {
          float v[8][kPer], wt[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {  // the group's loads first (8 rows in flight) ...
            const int s = sb + u;
            wt[u] = 0.f;
            if (s < s1) {
              const int64_t prow = (int64_t)pv.list_slot[s] * p.T_slot + r;
              wt[u] = __expf(__ldcg(p.part_lse + prow) - m);  // 0 for an empty partial
              const float* src = p.part_o + prow * D + lane * kPer;
#pragma unroll
              for (int j = 0; j < kPer; ++j) v[u][j] = __ldcg(src + j);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {  // ... then the fold in slot order
            if (sb + u < s1) {
              tot += wt[u];
#pragma unroll
              for (int j = 0; j < kPer; ++j) acc[j] = fmaf(wt[u], v[u][j], acc[j]);
            }
          }
        }
      }
      const float inv = tot > 0.f ? 1.f / tot : 0.f;
#pragma unroll
      for (int j = 0; j < kPer; ++j) acc[j] *= inv;
      const float lse = tot > 0.f ? m + __logf(tot) : -INFINITY;
      const int f = qt * pv.T_q + r;
      const int tok = f / p.g, head = kvh * p.g + f % p.g;
      const int64_t orow = (lm.qo_begin + tok) * (int64_t)p.H_qo + head;
      if (p.o_f32) {
        float* dst = reinterpret_cast<float*>(p.o) + orow * D + lane * kPer;
#pragma unroll
        for (int j = 0; j < kPer; ++j) dst[j] = acc[j];
      } else {
        TO* dst = reinterpret_cast<TO*>(p.o) + orow * D + lane * kPer;
#pragma unroll
        for (int j = 0; j < kPer; ++j) dst[j] = from_float<TO>(acc[j]);
      }
      if (p.lse && lane == 0) p.lse[orow] = lse;
    }
  }
  asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nthr) : "memory");  // s_flag reuse
}

template <typename TO, int D>
__device__ __forceinline__ void fused_contraction(const AttnParams& p, const PlanView& pv, int slot, int tid, int nthr,
                                                  int bar_id, volatile int* s_flag) {
  fused_contraction_meta<TO, D>(p, pv, nullptr, slot, tid, nthr, bar_id, s_flag);
}

// Standalone contraction (engines whose tiles can be 64/128/256 rows, where a merge list is too
// big for the one CTA that completes it): one warp per (list, row). Same closed form and the same
// operation order as fused_contraction (so the two placements are bitwise identical): the lanes
// read the slots' lse in parallel, form m = max and the weights w_s = e^{lse_s - m}; then the
// slots' rows are accumulated in plan order (R17) with 8 independent row loads in flight per
// warp (a dependent ⊕ chain would leave one load in flight and make the stage latency-bound).
template <typename TO, int D>
__global__ void __launch_bounds__(256) contraction_kernel(const __grid_constant__ AttnParams p) {
  // Latency-bound stage: the dependent global round trips per warp are plan header -> list
  // metadata -> (request, slot ids) -> every slot's lse AND o row (and the extra state) in one
  // round -> store. The o rows do not depend on the max, so groups of 8 slot rows are loaded
  // before m is known; the fold itself is the closed form in slot order (bitwise the same as
  // fused_contraction).
  constexpr int kPer = D / 32;
  constexpr int kGrp = 8;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const PlanView pv = load_plan(p.plan);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = (int64_t)pv.n_lists * pv.T_q;
  bool waited = false;  // PDL: the partials (and o) belong to the kernel before: wait once, late
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += nwarps) {
    const int li = (int)(w / pv.T_q), r = (int)(w % pv.T_q);
    const int req = pv.list_req[li], kvh = pv.list_kvh[li], qt = pv.list_qtile[li];
    const int s0 = pv.list_indptr[li], s1 = pv.list_indptr[li + 1];
    const int slot_l = s0 + lane < s1 ? pv.list_slot[s0 + lane] : 0;  // lane s: slot id of list entry s
    const int lq = pv.req_qo_len[req];
    const int64_t qo_begin = pv.req_qo_begin[req];
    const int f = qt * pv.T_q + r;
    if (f >= lq * p.g) continue;
    const int tok = f / p.g, head = kvh * p.g + f % p.g;
    const int64_t orow = (qo_begin + tok) * (int64_t)p.H_qo + head;
    const int ns = s1 - s0;
    if (!waited) {  // (a no-op without PDL) the plan / list reads above overlap the predecessor
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      waited = true;
    }
    // ---- one round of loads: lse of up to 32 slots (lane-parallel), o rows of the first group,
    // the extra state
    const float lse_l = lane < ns ? p.part_lse[(int64_t)slot_l * p.T_slot + r] : -INFINITY;
    float v[kGrp][kPer];
#pragma unroll
    for (int u = 0; u < kGrp; ++u) {
      const int sl = __shfl_sync(0xffffffffu, slot_l, u);
      if (u < ns) {
        const float* src = p.part_o + ((int64_t)sl * p.T_slot + r) * D + lane * kPer;
#pragma unroll
        for (int j = 0; j < kPer; ++j) v[u][j] = src[j];
      }
    }
    float xl = -INFINITY, xo[kPer];
    if (p.x_o) {
      xl = p.x_lse[orow];
      const float* src = p.x_o + orow * D + lane * kPer;
#pragma unroll
      for (int j = 0; j < kPer; ++j) xo[j] = src[j];
    }
    float m = lse_l;
    for (int s = s0 + 32 + lane; s < s1; s += 32)  // lists longer than a warp
      m = fmaxf(m, p.part_lse[(int64_t)pv.list_slot[s] * p.T_slot + r]);
    m = fmaxf(warp_max(m), xl);
    float acc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = 0.f;
    float tot = 0.f;
    if (m != -INFINITY) {
      for (int sb = 0; sb < ns; sb += kGrp) {
        float wt[kGrp];
        if (sb > 0) {  // later groups: their rows (the first group's are already in flight)
#pragma unroll
          for (int u = 0; u < kGrp; ++u) {
            if (sb + u < ns) {
              const int sl = pv.list_slot[s0 + sb + u];
              const float* src = p.part_o + ((int64_t)sl * p.T_slot + r) * D + lane * kPer;
#pragma unroll
              for (int j = 0; j < kPer; ++j) v[u][j] = src[j];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
          const int e = sb + u;
          float l = __shfl_sync(0xffffffffu, lse_l, e & 31);
          if (e >= 32 && e < ns) l = p.part_lse[(int64_t)pv.list_slot[s0 + e] * p.T_slot + r];
          wt[u] = e < ns ? __expf(l - m) : 0.f;  // 0 for an empty partial
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {  // the fold in slot order
          if (sb + u < ns) {
            tot += wt[u];
#pragma unroll
            for (int j = 0; j < kPer; ++j) acc[j] = fmaf(wt[u], v[u][j], acc[j]);
          }
        }
      }
      if (xl != -INFINITY) {
        const float wx = __expf(xl - m);
        tot += wx;
#pragma unroll
        for (int j = 0; j < kPer; ++j) acc[j] = fmaf(wx, xo[j], acc[j]);
      }
    }
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] *= inv;
    const float lse = tot > 0.f ? m + __logf(tot) : -INFINITY;
    store_row<TO, D>(p.o, orow, lane, acc, p.o_f32);
    if (p.lse && lane == 0) p.lse[orow] = lse;
  }
}

template <typename TI, typename TO, int D>
__global__ void __launch_bounds__(256) merge_states_kernel(const TI* __restrict__ oa, const float* __restrict__ la,
                                                           const TI* __restrict__ ob, const float* __restrict__ lb,
                                                           int64_t n, TO* out, float* lse_out) {
  constexpr int kPer = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t x = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); x < n; x += nwarps) {
    float acc[kPer], o[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      acc[j] = to_f<TI>(oa[x * D + lane * kPer + j]);
      o[j] = to_f<TI>(ob[x * D + lane * kPer + j]);
    }
    float l = la[x];
    // (o_a, lse_a) ⊕ (o_b, lse_b); identity when a is empty
    if (l == -INFINITY) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) acc[j] = lb[x] == -INFINITY ? 0.f : o[j];
      l = lb[x];
    } else {
      oplus<kPer>(acc, l, o, lb[x]);
    }
    __syncwarp();  // in-place: all lanes have read before anyone writes
#pragma unroll
    for (int j = 0; j < kPer; ++j) out[x * D + lane * kPer + j] = from_float<TO>(acc[j]);
    if (lse_out && lane == 0) lse_out[x] = l;
  }
}

template <typename TO, int D>
__global__ void __launch_bounds__(256) merge_many_kernel(const float* __restrict__ o_parts,
                                                         const float* __restrict__ lse_parts, int P, int64_t n,
                                                         TO* out, float* lse_out) {
  constexpr int kPer = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t x = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); x < n; x += nwarps) {
    float acc[kPer], l = -INFINITY;
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = 0.f;
    for (int q = 0; q < P; ++q) {
      float o[kPer];
      const float* src = o_parts + ((int64_t)q * n + x) * D + lane * kPer;
#pragma unroll
      for (int j = 0; j < kPer; ++j) o[j] = src[j];
      oplus<kPer>(acc, l, o, lse_parts[(int64_t)q * n + x]);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) out[x * D + lane * kPer + j] = from_float<TO>(acc[j]);
    if (lse_out && lane == 0) lse_out[x] = l;
  }
}

}  // namespace bsra
