// merge.cuh — the attention-state operator ⊕ (§2.2) on the GPU.
//
//  * contraction_kernel: the plan-driven "contraction" stage: for every merge
//    list (one per split (request, kv head, q tile)) fold ⊕ over its partial slots in the
//    plan's fixed order (ascending kv_begin, R17) — a left fold, no atomics on values
//    (P:240), so results are deterministic.
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

template <typename TO, int D>
__global__ void __launch_bounds__(256) contraction_kernel(const __grid_constant__ AttnParams p) {
  constexpr int kPer = D / 32;
  const PlanView pv = load_plan(p.plan);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = (int64_t)pv.n_lists * pv.T_q;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += nwarps) {
    const int li = (int)(w / pv.T_q), r = (int)(w % pv.T_q);
    const int req = pv.list_req[li], kvh = pv.list_kvh[li], qt = pv.list_qtile[li];
    const int lq = pv.req_qo_len[req];
    const int f = qt * pv.T_q + r;
    if (f >= lq * p.g) continue;
    const int tok = f / p.g, head = kvh * p.g + f % p.g;
    float acc[kPer], acc_lse = -INFINITY;
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = 0.f;
    for (int s = pv.list_indptr[li]; s < pv.list_indptr[li + 1]; ++s) {
      const int64_t prow = (int64_t)pv.list_slot[s] * p.T_slot + r;
      float o[kPer];
      const float* src = p.part_o + prow * D + lane * kPer;
#pragma unroll
      for (int j = 0; j < kPer; ++j) o[j] = src[j];
      oplus<kPer>(acc, acc_lse, o, p.part_lse[prow]);
    }
    const int64_t orow = (pv.req_qo_begin[req] + tok) * (int64_t)p.H_qo + head;
    store_row<TO, D>(p.o, orow, lane, acc, p.o_f32);
    if (p.lse && lane == 0) p.lse[orow] = acc_lse;
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
