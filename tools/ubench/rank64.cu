// slice_end_merge (expand_core.cuh) in isolation: one CTA of 288 threads, 8 warps' padded top-k
// lists in shared memory, clock64 around the rank merge per warp
#include <cstdio>
#include "expand_core.cuh"
using namespace smart;
__global__ void __launch_bounds__(288) rk(int k, unsigned long long* out, long long* cyc) {
  __shared__ ConsShared cs;
  __shared__ float2 msl[kMaxCpr * kConsumerWarps];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < kConsumerWarps * k) cs.cl[tid] = 0x8000000000000000ull + (unsigned long long)((tid * 7919u) % 1000u) * 4096 + tid;
  if (tid < 16 * 8) msl[tid] = make_float2(1.f, 2.f);
  __syncthreads();
  if (warp >= 8) return;
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    slice_end_merge(cs, msl, k, 2, [&](int rank, unsigned long long key) { out[rank + 32 * rep] = key; },
                    [&](int cc, float M, float S) { out[512 + cc] = __float_as_uint(M); });
    consumer_sync();
  }
  long long t1 = clock64();
  if ((tid & 31) == 0) cyc[warp] = (t1 - t0) / 10;
}
int main() {
  unsigned long long* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
  for (int k : {8, 10}) {
    for (int r = 0; r < 3; ++r) rk<<<1, 288>>>(k, o, c);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("k %d: slice_end_merge cycles per call (warps 0..7):", k);
    for (int w = 0; w < 8; ++w) printf(" %lld", h[w]);
    printf("  [%s]\n", cudaGetErrorString(cudaGetLastError()));
  }
}
