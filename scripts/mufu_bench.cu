// Microbenchmark: sustained MUFU.EX2 and FFMA2 throughput per SM on this GPU (ops/clk/SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/mufu_bench.cu -o /tmp/mufu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ex2_kernel(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma2_kernel(float* out, int iters, long long* cyc) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(0.001f * threadIdx.x, 0.002f * i);
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    long long h[148];
    ex2_kernel<<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 8;
    printf("ex2   threads %4d: %.2f ops/clk/SM\n", threads, ops / h[0]);
    ffma2_kernel<<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    printf("ffma2 threads %4d: %.2f instr/clk/SM (x2 flops lanes)\n", threads, ops / h[0]);
  }
  return 0;
}
