// fp8cvt_bench.cu — E4M3 -> bf16 conversion variants for the tc_decode converter warps:
// exactness over all 65536 byte pairs (against the f16 -> f32 -> bf16 reference) and throughput
// (16 warps per SM, each converting registers in a dependent-free unrolled loop).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/fp8cvt_bench.cu -o /tmp/fp8cvt && /tmp/fp8cvt
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdio>
#include <cstdint>

// (0) reference: cvt e4m3x2 -> f16x2, f16 -> f32, f32x2 -> bf16x2
__device__ __forceinline__ void cvt_ref(uint32_t w, uint32_t& lo, uint32_t& hi) {
  uint32_t r[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const __half2_raw x = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w >> (16 * h)), __NV_E4M3);
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&x));
    const __nv_bfloat162 b = __float22bfloat162_rn(f);
    r[h] = *reinterpret_cast<const uint32_t*>(&b);
  }
  lo = r[0];
  hi = r[1];
}
// (1) ALU: bf16 bits of value * 2^-120 by shifts/masks, HMUL2.BF16 by 2^120, PRMT un-permute
__device__ __forceinline__ void cvt_alu(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t a = (w & 0x80008000u) | ((w >> 4) & 0x07F007F0u);         // (b1, b3)
  const uint32_t b = ((w << 8) & 0x80008000u) | ((w << 4) & 0x07F007F0u);  // (b0, b2)
  const uint32_t sb = 0x7B807B80u;  // bf16x2 (2^120, 2^120)
  const __nv_bfloat162 s = *reinterpret_cast<const __nv_bfloat162*>(&sb);
  __nv_bfloat162 A = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&a), s);
  __nv_bfloat162 B = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&b), s);
  const uint32_t ua = *reinterpret_cast<uint32_t*>(&A), ub = *reinterpret_cast<uint32_t*>(&B);
  lo = __byte_perm(ub, ua, 0x5410);  // (b0, b1)
  hi = __byte_perm(ub, ua, 0x7632);  // (b2, b3)
}
// (2) f16 unpack (exact, all normal or zero) then bf16 bits of value * 2^-112, HMUL2.BF16 by 2^112
__device__ __forceinline__ void cvt_f16(uint32_t w, uint32_t& lo, uint32_t& hi) {
  uint32_t r[2];
  const uint32_t sb = 0x77807780u;  // bf16x2 (2^112, 2^112)
  const __nv_bfloat162 s = *reinterpret_cast<const __nv_bfloat162*>(&sb);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const __half2_raw x = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w >> (16 * h)), __NV_E4M3);
    const uint32_t u = (uint32_t)x.x | ((uint32_t)x.y << 16);
    const uint32_t t = (u & 0x80008000u) | ((u >> 3) & 0x0FFF0FFFu);
    __nv_bfloat162 B = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&t), s);
    r[h] = *reinterpret_cast<uint32_t*>(&B);
  }
  lo = r[0];
  hi = r[1];
}
// (3) f16 output only (the f16-q variant)
__device__ __forceinline__ void cvt_half(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const __half2_raw x = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)w, __NV_E4M3);
  const __half2_raw y = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w >> 16), __NV_E4M3);
  lo = (uint32_t)x.x | ((uint32_t)x.y << 16);
  hi = (uint32_t)y.x | ((uint32_t)y.y << 16);
}

template <int V>
__device__ __forceinline__ void cvt(uint32_t w, uint32_t& lo, uint32_t& hi) {
  if (V == 0) cvt_ref(w, lo, hi);
  if (V == 1) cvt_alu(w, lo, hi);
  if (V == 2) cvt_f16(w, lo, hi);
  if (V == 3) cvt_half(w, lo, hi);
}

template <int V>
__global__ void check(uint32_t* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // 2^16 pairs x 2 orders
  if (i >= 65536) return;
  const uint32_t w = i | ((65535u - i) << 16);
  uint32_t lo, hi, rl, rh;
  cvt<V>(w, lo, hi);
  cvt_ref(w, rl, rh);
  // NaN codes 0x7F / 0xFF: compare only non-NaN outputs
  for (int k = 0; k < 4; ++k) {
    const uint32_t byte = (w >> (8 * k)) & 0xFF;
    if ((byte & 0x7F) == 0x7F) continue;
    const uint32_t got = ((k < 2 ? lo : hi) >> (16 * (k & 1))) & 0xFFFF;
    const uint32_t ref = ((k < 2 ? rl : rh) >> (16 * (k & 1))) & 0xFFFF;
    if (got != ref) atomicAdd(bad, 1u);
  }
}

template <int V>
__global__ void bench(const uint4* in, uint4* out, int iters) {
  uint4 u = in[threadIdx.x & 31];
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t lo, hi;
      cvt<V>(w[i], lo, hi);
      acc ^= lo + hi;
    }
    u.x += acc;  // loop-carried dependence keeps every word's conversion live
    u.y ^= acc;
    u.z += acc << 1;
    u.w ^= acc >> 3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = make_uint4(acc, 0, 0, 0);
}

template <int V>
void run(const char* name, uint32_t* d_bad, const uint4* d_in, uint4* d_out, int sms) {
  cudaMemset(d_bad, 0, 4);
  check<V><<<256, 256>>>(d_bad);
  uint32_t bad = 0;
  cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost);
  const int iters = 4096, threads = 512;
  bench<V><<<sms, threads>>>(d_in, d_out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<V><<<sms, threads>>>(d_in, d_out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double elems = (double)sms * threads * iters * 16;
  const double per_clk_sm = elems / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("{\"variant\": \"%s\", \"mismatches\": %u, \"elems_per_clk_per_sm\": %.1f}\n", name, bad, per_clk_sm);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d_bad;
  uint4 *d_in, *d_out;
  cudaMalloc(&d_bad, 4);
  cudaMalloc(&d_in, 32 * 16);
  cudaMalloc(&d_out, (size_t)sms * 512 * 16);
  cudaMemset(d_in, 0x3A, 32 * 16);
  run<0>("ref_cvt_f16_f32_bf16", d_bad, d_in, d_out, sms);
  run<1>("alu_shift_hmul2_prmt", d_bad, d_in, d_out, sms);
  run<2>("cvt_f16_then_alu_hmul2", d_bad, d_in, d_out, sms);
  run<3>("cvt_f16_only", d_bad, d_in, d_out, sms);
  return 0;
}
