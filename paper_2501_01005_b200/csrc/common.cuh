// common.cuh — kernel parameter block and device-side view of the plan image.
//
// The plan image (scheduler.cpp) lives in a fixed workspace section (App. D.1); kernels
// read its header at run time, so one captured CUDA graph stays valid across re-plans.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

namespace bsra {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnParams {
  const int32_t* plan;  // device plan image
  const void* q;
  const void* k;
  const void* v;
  int64_t ks0, ks1, ks2;  // k_pool strides (elements): page, token, head
  int64_t vs0, vs1, vs2;
  const int32_t* page_indices;
  const uint8_t* mask;
  const int64_t* mask_indptr;
  void* o;
  float* lse;
  float* part_o;    // [slots][T_slot][D] fp32
  float* part_lse;  // [slots][T_slot]
  int32_t* counters;  // per-merge-list arrival counters (fused contraction)
  long long* trace;   // optional pipeline trace (CTA 0 event clocks), NULL in production
  int32_t fused_merge;  // 1: split items are merged in-kernel (decode engines); 0: contraction kernel
  // 1: contiguous (ragged) KV: token t of request i is row page_begin_i + t of
  // k/v [N, H_kv, D] (page_begin = kv_indptr[i]); no page table. The tcgen05 kernels address it
  // through a pool map whose token dimension is N (TMA clips at the buffer end).
  int32_t kv_ragged;
  // Attention variants (R26 / R27), 0 = off. window: sliding window W, a
  // row at position p hides keys t < p - W + 1. soft_cap: c / sm_scale, the cap in raw q.k units,
  // so the transformed raw score cap * tanh(s / cap) goes through the same scale-and-exp path.
  int32_t window;
  float soft_cap, inv_soft_cap;
  int32_t H_qo, H_kv, g, page_size, mask_mode, o_f32, T_slot, D;
  float scale_log2;  // sm_scale * log2(e) (fp8 KV: sm_scale * k_scale * log2(e))
  // fp8 KV cache (R28): pools hold E4M3 bytes; v_scale multiplies o
  int32_t kv_f8;
  float v_scale;
  // ALiBi (R30): raw score s += slope_h / logit_scale * (t - p)
  int32_t alibi;
  float inv_logit_scale;
  // RoPE (P:228 / P:329-338, R31): pair (i, i + D/2) turns by pos * theta_i; rope_f[i] =
  // theta_i / 2pi as a 0.64 fixed-point fraction of a turn, so (pos * rope_f[i]) mod 2^64 is the
  // angle's fraction of a turn, exact for every position
  int32_t rope;
  uint64_t rope_f[64];
  // contraction kernel only (bsra_contract): an extra state ⊕-combined into every folded row
  const float* x_o;    // [rows, H_qo, D] fp32, the layout of o; NULL = none
  const float* x_lse;  // [rows, H_qo]
};

// sin / cos of the RoPE angle pos * theta (frequency f = theta / 2pi in 2^-64 turns): the 64-bit
// product wraps modulo one turn exactly, its top 32 bits (signed) are the angle in [-pi, pi) to
// 2^-31 of a turn, and __sincosf is accurate to ~2^-21 on that range (no large-argument loss).
__device__ __forceinline__ void rope_sincos(int64_t pos, uint64_t f, float& sn, float& cs) {
  const uint64_t u = (uint64_t)pos * f;
  const float a = (float)(int32_t)(u >> 32) * 1.4629180792671596e-09f;  // 2pi / 2^32
  __sincosf(a, &sn, &cs);
}
// The same angle through the correctly rounded sincosf (for constants a recurrence reuses)
__device__ __forceinline__ void rope_sincos_precise(int64_t pos, uint64_t f, float& sn, float& cs) {
  const uint64_t u = (uint64_t)pos * f;
  sincosf((float)(int32_t)(u >> 32) * 1.4629180792671596e-09f, &sn, &cs);
}

// LogitsTransform soft-cap on a raw score (R27): s -> c * tanh(s / c), c in raw units.
// tanh x = 1 - 2 / (2^(2x log2 e) + 1): one ex2 and one rcp (absolute error ~1e-7, i.e. ~c*1e-7
// in the logit; tanh.approx.f32's 2^-11 relative error would exceed the lse tolerance at c = 50).
// Saturates correctly: x -> +inf gives 1, x -> -inf gives -1.
__device__ __forceinline__ float soft_cap_raw(const AttnParams& p, float s) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(s * p.inv_soft_cap * 2.8853900817779268f));  // 2 log2(e)
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.f));
  return p.soft_cap * fmaf(-2.f, r, 1.f);
}

// ALiBi slope of qo head h of H in raw q.k units (R30); fp64 once per row for a correctly
// rounded slope (n = 2^floor(log2 H); h < n: 2^(-8(h+1)/n), else 2^(-4(2(h-n)+1)/n))
__device__ __forceinline__ float alibi_slope_raw(const AttnParams& p, int h) {
  const int n = 1 << (31 - __clz(p.H_qo));
  const double e = h < n ? -8.0 * (h + 1) / n : -4.0 * (2 * (h - n) + 1) / n;
  return (float)(exp2(e) * (double)p.inv_logit_scale);
}

struct PlanView {
  int32_t num_ctas, T_q, L, n_items, n_lists, n_slots, batch, g, H_kv, mask;
  const int32_t* cta_indptr;
  const int32_t* item_req;
  const int32_t* item_kvh;
  const int32_t* item_qtile;
  const int32_t* item_kb;
  const int32_t* item_ke;
  const int32_t* item_slot;
  const int32_t* list_indptr;
  const int32_t* list_slot;
  const int32_t* list_req;
  const int32_t* list_kvh;
  const int32_t* list_qtile;
  const int32_t* req_qo_begin;
  const int32_t* req_qo_len;
  const int32_t* req_kv_len;
  const int32_t* req_page_begin;
};

__device__ __forceinline__ PlanView load_plan(const int32_t* __restrict__ p) {
  PlanView v;
  v.num_ctas = p[2];
  v.T_q = p[3];
  v.L = p[4];
  v.n_items = p[5];
  v.n_lists = p[6];
  v.n_slots = p[7];
  v.batch = p[8];
  v.g = p[9];
  v.H_kv = p[10];
  v.mask = p[11];
  const int32_t* c = p + 16;
  v.cta_indptr = c;
  c += v.num_ctas + 1;
  v.item_req = c;
  c += v.n_items;
  v.item_kvh = c;
  c += v.n_items;
  v.item_qtile = c;
  c += v.n_items;
  v.item_kb = c;
  c += v.n_items;
  v.item_ke = c;
  c += v.n_items;
  v.item_slot = c;
  c += v.n_items;
  v.list_indptr = c;
  c += v.n_lists + 1;
  v.list_slot = c;
  c += v.n_slots;
  v.list_req = c;
  c += v.n_lists;
  v.list_kvh = c;
  c += v.n_lists;
  v.list_qtile = c;
  c += v.n_lists;
  v.req_qo_begin = c;
  c += v.batch;
  v.req_qo_len = c;
  c += v.batch;
  v.req_kv_len = c;
  c += v.batch;
  v.req_page_begin = c;
  return v;
}

// ---- element conversions (16-byte vectors)
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void to_float(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void to_float(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};
template <>
struct Vec<__half> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void to_float(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 x = __half22float2(h);
      f[2 * i] = x.x;
      f[2 * i + 1] = x.y;
    }
  }
};

// OCP E4M3 (R28): 16 bytes -> 16 floats via the exact fp8x2 -> f16x2 converter
template <>
struct Vec<__nv_fp8_e4m3> {
  static constexpr int N = 16;
  __device__ __forceinline__ static void to_float(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const __half2_raw r = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[i] >> (16 * h)), __NV_E4M3);
        const float2 x = __half22float2(*reinterpret_cast<const __half2*>(&r));
        f[4 * i + 2 * h] = x.x;
        f[4 * i + 2 * h + 1] = x.y;
      }
    }
  }
};

template <typename T>
__device__ __forceinline__ T from_float(float x);
template <>
__device__ __forceinline__ float from_float<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_float<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <>
__device__ __forceinline__ __half from_float<__half>(float x) { return __float2half_rn(x); }

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <>
__device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }
template <>
__device__ __forceinline__ float to_f<__nv_fp8_e4m3>(__nv_fp8_e4m3 x) { return float(x); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// 16-byte cp.async with zero fill: src_bytes = 0 writes 16 zero bytes and reads nothing
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
// arrive on an mbarrier once all of this thread's prior cp.async copies have completed (the
// barrier's expected count includes this arrival: .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// custom-mask bit (R9): row-major l_qo x l_kv per request, LSB first
__device__ __forceinline__ bool mask_bit(const uint8_t* __restrict__ m, int64_t j) {
  return (__ldg(m + (j >> 3)) >> (j & 7)) & 1;
}

}  // namespace bsra
