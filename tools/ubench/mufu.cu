// MUFU.EX2 / FFMA2 throughput microbenchmark (debug aid): results per clock per SM
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int n, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-6f;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f33800000;" : "+f"(a[i]));
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
int main() {
  float* o; cudaMalloc(&o, 148 * 1024 * 4 * 8);
  const int n = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (int thr : {256, 512, 1024}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      if (mode == 0) k<0><<<148, thr>>>(o, n, 1.f); else k<1><<<148, thr>>>(o, n, 1.f);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) { if (mode == 0) k<0><<<148, thr>>>(o, n, 1.f); else k<1><<<148, thr>>>(o, n, 1.f); }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      float cyc; cudaMemcpy(&cyc, o, 4, cudaMemcpyDeviceToHost);
      double ops = (double)thr * n * 8;  // per SM
      printf("%s threads/SM %4d: %.1f ops/clk/SM (clock64), %.3f Tops/s total\n", mode == 0 ? "ex2 " : "ffma", thr, ops / cyc, ops * 148 / (ms / 1e3) / 1e12);
    }
  return 0;
}
