// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM on this GPU (ops per clock per SM).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void k_ex2(float* out, int iters, long long* clk) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ex2(a[i]) - 1.0f;
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float* out, int iters, long long* clk) {
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  const float2 b = make_float2(0.999f, 0.999f), c = make_float2(1e-3f, 1e-3f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk; cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&clk, sms * 8);
  long long h[1024];
  for (int threads : {128, 256, 512, 1024}) {
    const int iters = 4096;
    k_ex2<<<sms, threads>>>(out, iters, clk); cudaDeviceSynchronize();
    k_ex2<<<sms, threads>>>(out, iters, clk); cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 8;
    printf("ex2   threads/SM %4d: %.2f ops/clk/SM\n", threads, ops / h[0]);
    k_ffma2<<<sms, threads>>>(out, iters, clk); cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost);
    printf("ffma2 threads/SM %4d: %.2f fp32 ops(2 per FFMA2 lane)/clk/SM\n", threads, ops * 2 / h[0]);
  }
  return 0;
}
