// Standalone check of the 5-D page-box view used by tc_decode kGrp: one TMA box of an NHD pool page
// lands as [token group][64-column half][8 rows][128 B] (SW128); a c dimension of 2^32 - 1 encodes
// but traps at run time (arg 0 vs 1). nvcc -gencode arch=compute_100a,code=sm_100a scripts/tma5d_layout_check.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int c3, int c4, uint16_t* out) {
  __shared__ __align__(1024) uint8_t sm[4096 + 1024];
  __shared__ uint64_t bar;
  uint8_t* s = sm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(4096) : "memory");
    if (c3 >= 0)
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n"
                 ::"r"(su32(s)), "l"(&tm), "r"(su32(&bar)), "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4) : "memory");
    else {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n"
                 ::"r"(su32(s)), "l"(&tm), "r"(su32(&bar)), "r"(0), "r"(0), "r"(0), "r"(c4) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n"
                 ::"r"(su32(s + 2048)), "l"(&tm), "r"(su32(&bar)), "r"(0), "r"(-c3 == 1 ? 8 : 0), "r"(0), "r"(c4) : "memory");
    }
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(&bar)), "r"(0) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(s)[i];
}
int main(int argc, char** argv) {
  const int var = argc > 1 ? atoi(argv[1]) : 0;
  const int P = 4, PS = 16, H = 8, D = 128;
  std::vector<uint16_t> h((size_t)P * PS * H * D);
  for (int p = 0; p < P; ++p) for (int t = 0; t < PS; ++t) for (int hh = 0; hh < H; ++hh) for (int d = 0; d < D; ++d)
    h[(((size_t)p * PS + t) * H + hh) * D + d] = (uint16_t)((p << 13) | (t << 9) | (hh << 7) | d);
  void* g; cudaMalloc(&g, h.size() * 2); cudaMemcpy(g, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  uint16_t* out; cudaMalloc(&out, 4096);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
  const long s0 = PS * H * D, s1 = H * D, s2 = D;
  CUtensorMap tm;
  cuuint64_t dims[5] = {64, 8, 2, (cuuint64_t)(PS / 8), var & 1 ? (cuuint64_t)(P * (s0 / s2)) : 0x7fffffffull};
  cuuint64_t strides[4] = {(cuuint64_t)s1 * 2, 128, (cuuint64_t)s1 * 16, (cuuint64_t)s2 * 2};
  cuuint32_t box[5] = {64, 8, 2, 2, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (var & 2) {  // 4-D: (d_lo, tok 16, half, c) box (64, 8, 2, 1): tok dim contiguous-ish
    cuuint64_t d4[4] = {64, (cuuint64_t)PS, 2, dims[4]};
    cuuint64_t s4[3] = {(cuuint64_t)s1 * 2, 128, (cuuint64_t)s2 * 2};
    cuuint32_t b4[4] = {64, 8, 2, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, g, d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (var & 4) {  // monotonic strides: (d_lo, half, tok, c): smem [tok][half] -- layout check will fail, only tests legality
    cuuint64_t d4[4] = {64, 2, (cuuint64_t)PS, dims[4]};
    cuuint64_t s4[3] = {128, (cuuint64_t)s1 * 2, (cuuint64_t)s2 * 2};
    cuuint32_t b4[4] = {64, 2, 16, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, g, d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("var %d encode %d\n", var, (int)r);
  const int page = 2, head = 3, cs = s0 / s2;
  k<<<1, 128>>>(tm, (var & 6) ? -1 : 0, page * cs + head, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> o(2048); cudaMemcpy(o.data(), out, 4096, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int grp = 0; grp < 2; ++grp) for (int half = 0; half < 2; ++half) for (int r8 = 0; r8 < 8; ++r8) for (int c = 0; c < 8; ++c) {
    // smem 16B chunk c of row (grp, half, r8) holds logical chunk c ^ r8 (SW128)
    const int base = ((grp * 2 + half) * 8 + r8) * 64 + c * 8;
    const int lc = c ^ r8;
    const int tok = grp * 8 + r8;
    for (int e2 = 0; e2 < 8; ++e2) {
      const int d = half * 64 + lc * 8 + e2;
      const uint16_t want = (uint16_t)((page << 13) | (tok << 9) | (head << 7) | d);
      if (o[base + e2] != want) { if (bad < 5) printf("mismatch grp %d half %d row %d chunk %d: got %x want %x\n", grp, half, r8, c, o[base+e2], want); ++bad; }
    }
  }
  printf("bad = %d\n", bad);
  return 0;
}
