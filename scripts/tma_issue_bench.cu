// Microbenchmark: TMA tiled-load issue throughput per SM (one CTA per SM, 148 CTAs) as a function
// of the box size (rows of 128 B, SWIZZLE_128B, the decode kernel's page boxes), the number of
// issuing warps and lanes, with the source resident in L2 (32 MB) or streamed from HBM (1 GB).
// Each issuing warp owns a ring of 4 stages x 16 KB; a stage's boxes complete on one mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/tma_issue_bench.cu -o /tmp/tmab -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows,
                                                    int warps, int lanes, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kStages = 4, kStageBytes = 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + warps * kStages * kStageBytes);
  if (threadIdx.x < warps * kStages)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  __syncthreads();
  const int box_bytes = box_rows * 128;
  const int per_stage = kStageBytes / box_bytes;  // boxes per stage
  long long t0 = clock64();
  if (warp < warps) {
    uint32_t ph[kStages] = {0, 0, 0, 0};
    unsigned h = blockIdx.x * 7919u + warp * 104729u;
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      uint64_t* b = &bar[warp * kStages + s];
      if (it >= kStages) {  // wait for this stage's previous fill
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                       : "=r"(ok) : "r"(su32(b)), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
      }
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(kStageBytes) : "memory");
      __syncwarp();
      uint8_t* dst = smem + (warp * kStages + s) * kStageBytes;
      for (int j0 = 0; j0 < per_stage; j0 += lanes) {
        const int j = j0 + lane;
        if (lane < lanes && j < per_stage) {
          h = h * 1664525u + 1013904223u;
          const int row = (int)((h >> 8) % (unsigned)(rows_total / box_rows)) * box_rows;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                  su32(dst + j * box_bytes)),
              "l"(&tm), "r"(su32(b)), "r"((j & 1) * 64), "r"(row)
              : "memory");
        }
      }
      __syncwarp();
    }
    for (int s = 0; s < kStages; ++s) {  // drain
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(ok) : "r"(su32(&bar[warp * kStages + s])), "r"(ph[s]) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  CUtensorMap tm;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  long long h[148];
  for (size_t mb : {32, 1024}) {
    const size_t bytes = mb << 20;
    void* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    const int rows = (int)(bytes / 256);  // rows of 128 bf16 (256 B); a box takes 64 columns
    for (int box_rows : {4, 16, 32}) {
      cuuint64_t dims[2] = {128, (cuuint64_t)rows};
      cuuint64_t strides[1] = {256};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
      }
      for (int warps : {1, 2, 3}) {
        for (int lanes : {8, 32}) {
          const int iters = 64;
          const int smem = warps * 4 * 16384 + 1024 + 256;
          if (smem > 227 * 1024) continue;
          cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          // each box instruction moves box_rows x 128 B (one 64-column half)
          tma_kernel<<<148, 128, smem>>>(tm, rows, box_rows, warps, lanes, 4, cyc);
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          cudaEventRecord(a);
          tma_kernel<<<148, 128, smem>>>(tm, rows, box_rows, warps, lanes, iters, cyc);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
          long long mx = 0;
          for (long long x : h) mx = x > mx ? x : mx;
          const double ops = (double)warps * iters * (16384.0 / (box_rows * 128));
          const double gbs = 148.0 * warps * iters * 16384.0 / (ms * 1e-3) / 1e9;
          printf("{\"src_MB\": %zu, \"box_rows\": %d, \"box_bytes\": %d, \"warps\": %d, \"lanes\": %d, \"cyc_per_op\": %.1f, "
                 "\"B_per_clk_SM\": %.1f, \"GB_s_total\": %.0f, \"err\": \"%s\"}\n",
                 mb, box_rows, box_rows * 128, warps, lanes, mx / ops, ops * box_rows * 128 / mx, gbs,
                 cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
    cudaFree(src);
  }
  return 0;
}
