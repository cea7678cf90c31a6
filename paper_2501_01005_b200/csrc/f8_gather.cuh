// f8_gather.cuh — fp8 KV cache for the prefill tiles (T_q >= 64): dequantise-and-gather pass.
//
// The paper's mixed-precision attention keeps q / o in 16 bits and the KV cache in fp8
// (App. F). Prefill is tensor-bound (every K/V tile feeds 128-256 query rows), so
// here the dequantisation runs as one HBM-bound pass ahead of the 16-bit prefill kernel instead
// of inside it: every token the plan covers is read once from the E4M3 pool (through the BSR page
// table, or from a contiguous KV) and written as 16-bit rows [sum l_kv, H_kv, 128] in request
// order into an engine-owned buffer; the tcgen05 prefill kernel then runs on it as contiguous
// KV (BSRA_FLAG_RAGGED_KV addressing). Extra HBM traffic is 1 B read + 2 B written
// per element, once per run() — about 3 % of configs[2]'s prefill time.
// The per-tensor k_scale / v_scale stay in the attention kernel (logit scale and o), so the
// 16-bit rows hold the E4M3 values exactly.
//
// One warp per token row (H_kv * 128 bytes); grid-stride over the plan's tokens, so a graph
// captured once serves every re-plan (the token count and offsets are read from the device).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <cstdint>

namespace bsra {

struct F8GatherParams {
  const uint8_t* k;
  const uint8_t* v;
  int64_t ks0, ks1, ks2, vs0, vs1, vs2;  // element (= byte) strides: page, slot, head
  const int32_t* page_indices;           // BSR indices (paged source), NULL for contiguous
  const int32_t* src_begin;              // [batch+1]: kv_page_indptr (paged) or kv_indptr (contiguous)
  const int32_t* kv_off;                 // [batch+1]: first destination row of each request
  const int32_t* plan;                   // plan image (header word 8 = batch)
  int32_t page_size, H_kv, f16;
  uint16_t* ko;                          // [kv_off[batch], H_kv, 128] 16-bit
  uint16_t* vo;
};

// 16 E4M3 bytes -> 16 bf16 / f16 values in natural order (exact: cvt to f16x2, then f32 -> bf16)
__device__ __forceinline__ void f8g_convert16(const uint4& u, bool f16, uint4& lo, uint4& hi) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const __half2_raw x = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[i] >> (16 * h)), __NV_E4M3);
      if (f16) {
        r[2 * i + h] = (uint32_t)x.x | ((uint32_t)x.y << 16);
      } else {
        const __nv_bfloat162 b = __float22bfloat162_rn(__half22float2(*reinterpret_cast<const __half2*>(&x)));
        r[2 * i + h] = *reinterpret_cast<const uint32_t*>(&b);
      }
    }
  }
  lo = make_uint4(r[0], r[1], r[2], r[3]);
  hi = make_uint4(r[4], r[5], r[6], r[7]);
}

__global__ void __launch_bounds__(256) f8_gather_kernel(const __grid_constant__ F8GatherParams g) {
  const int batch = g.plan[8];
  if (batch <= 0) return;
  const int64_t total = g.kv_off[batch];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int chunks = g.H_kv * 8;  // 16-byte fp8 chunks per token row
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < total; row += nwarps) {
    int lo = 0, hi = batch;  // request i with kv_off[i] <= row < kv_off[i+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(g.kv_off + mid) <= row) lo = mid;
      else hi = mid;
    }
    const int64_t t = row - __ldg(g.kv_off + lo);
    int64_t page, slot;
    if (g.page_indices) {
      page = __ldg(g.page_indices + __ldg(g.src_begin + lo) + t / g.page_size);
      slot = t % g.page_size;
    } else {
      page = 0;
      slot = __ldg(g.src_begin + lo) + t;
    }
    for (int c = lane; c < chunks; c += 32) {
      const int h = c >> 3, j = c & 7;
      const uint4 uk = __ldg(reinterpret_cast<const uint4*>(g.k + page * g.ks0 + slot * g.ks1 + h * g.ks2) + j);
      const uint4 uv = __ldg(reinterpret_cast<const uint4*>(g.v + page * g.vs0 + slot * g.vs1 + h * g.vs2) + j);
      uint4 a, b;
      uint4* dk = reinterpret_cast<uint4*>(g.ko + (row * g.H_kv + h) * 128 + j * 16);
      uint4* dv = reinterpret_cast<uint4*>(g.vo + (row * g.H_kv + h) * 128 + j * 16);
      f8g_convert16(uk, g.f16 != 0, a, b);
      dk[0] = a;
      dk[1] = b;
      f8g_convert16(uv, g.f16 != 0, a, b);
      dv[0] = a;
      dv[1] = b;
    }
  }
}

}  // namespace bsra
