// latency microbenchmark (debug aid): one warp, dependent chains of common ops
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out, int n, const unsigned long long* g) {
  __shared__ unsigned long long s[1024];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 3) & 1023;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  unsigned long long t0, t1;
  // (a) dependent LDS chain
  unsigned long long x = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = s[x & 1023];
  t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / n;
  // (b) independent LDS, 2 accumulators
  int r0 = 0, r1 = 0;
  unsigned long long key = s[lane] + x;
  t0 = clock64();
  for (int i = 0; i + 1 < n; i += 2) {
    r0 += s[i & 1023] > key;
    r1 += s[(i + 1) & 1023] > key;
  }
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0) / n + (r0 + r1 == 12345);
  // (c) dependent SHFL
  int v = lane + (int)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (v + i) & 31);
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0) / n + (v == 12345);
  // (d) dependent VOTE+POPC
  int w = lane + (int)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) w += __popc(__ballot_sync(0xffffffffu, (w & 1)));
  t1 = clock64();
  if (lane == 0) out[3] = (t1 - t0) / n + (w == 12345);
  // (e) dependent REDUX
  unsigned u = lane + (unsigned)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + lane);
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0) / n + (u == 12345);
  // (f) dependent IADD chain
  int a = lane + (int)x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) a = a * 3 + i;
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0) / n + (a == 12345);
  // (g) dependent global load chain (L2/L1)
  unsigned long long y = lane;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) y = __ldcg(&g[y & 4095]);
  t1 = clock64();
  if (lane == 0) out[6] = (t1 - t0) / 64 + (y == 12345);
  // (h) double add chain
  double d = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) d = d * 1.0000001 + 0.5;
  t1 = clock64();
  if (lane == 0) out[7] = (t1 - t0) / n + (d == 12345.0);
  // (i) double shfl
  t0 = clock64();
  for (int i = 0; i < n; ++i) d = __shfl_xor_sync(0xffffffffu, d, 1) + 1.0;
  t1 = clock64();
  if (lane == 0) out[8] = (t1 - t0) / n + (d == 12345.0);
  // (j) named barrier with 1 warp
  t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 32;");
  t1 = clock64();
  if (lane == 0) out[9] = (t1 - t0) / n;
  // (k) clock64 overhead
  t0 = clock64();
  for (int i = 0; i < n; ++i) { unsigned long long c = clock64(); a += (int)c; }
  t1 = clock64();
  if (lane == 0) out[10] = (t1 - t0) / n + (a == 12345);
  // (l) double division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) d = 3.0 / (d + 1.0);
  t1 = clock64();
  if (lane == 0) out[11] = (t1 - t0) / n + (d == 12345.0);
  // (m) float division chain
  float f = lane + 1.f;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = 3.f / (f + 1.f);
  t1 = clock64();
  if (lane == 0) out[12] = (t1 - t0) / n + (f == 12345.f);
  // (n) smem atomicOr
  __shared__ unsigned bm[64];
  if (lane < 64) bm[lane] = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) atomicOr(&bm[(lane + i) & 63], 1u << (i & 31));
  t1 = clock64();
  if (lane == 0) out[13] = (t1 - t0) / n;
  // (o) F2F f32->f64 + DMUL dep
  float q = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = (float)((double)q * 1.0000001);
  t1 = clock64();
  if (lane == 0) out[14] = (t1 - t0) / n + (q == 12345.f);
}
int main() {
  unsigned long long *o, *g, h[16] = {};
  cudaMalloc(&o, 16 * 8);
  cudaMalloc(&g, 4096 * 8);
  unsigned long long hg[4096];
  for (int i = 0; i < 4096; ++i) hg[i] = (i * 131 + 7) & 4095;
  cudaMemcpy(g, hg, sizeof hg, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) k<<<1, 288>>>(o, 256, g);
  cudaDeviceSynchronize();
  cudaMemcpy(h, o, 16 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"LDS dep", "LDS indep/elem", "SHFL dep", "VOTE+POPC dep", "REDUX dep", "IMAD dep",
                      "LDG.cg dep (L2)", "DFMA dep", "SHFL.f64+DADD dep", "BAR 1 warp", "CS2R clock", "DDIV dep", "FDIV dep", "ATOMS.OR", "F2F+DMUL+F2F dep"};
  for (int i = 0; i < 15; ++i) printf("%-22s %llu cycles\n", nm[i], h[i]);
  return 0;
}
