// Round latency of the selection tournament (select_core.cuh select_tournament): one warp pops
// 32 winners from 32 sorted lists of 8 keys in shared memory; variants of the warp min.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench/tourn.cu -o /tmp/tourn
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned redux_min(unsigned v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ unsigned shfl_min(unsigned v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int MODE>
__global__ void tourn(const unsigned long long* gkeys, unsigned long long* out, long long* cyc, int rounds) {
  __shared__ unsigned long long keys[32 * 8];
  __shared__ unsigned long long win[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < 256; i += 32) keys[i] = gkeys[i];
  __syncwarp();
  unsigned long long cur = keys[lane * 8], nxt = keys[lane * 8 + 1];
  int h = 0;
  long long t0 = clock64();
  for (int j = 0; j < rounds; ++j) {
    unsigned hi;
    if (MODE == 1) hi = shfl_min((unsigned)(cur >> 32));
    else hi = redux_min((unsigned)(cur >> 32));
    unsigned bal = __ballot_sync(0xffffffffu, (unsigned)(cur >> 32) == hi);
    if (__popc(bal) > 1) {
      const unsigned lo = redux_min((unsigned)(cur >> 32) == hi ? (unsigned)cur : 0xffffffffu);
      bal = __ballot_sync(0xffffffffu, (unsigned)(cur >> 32) == hi && (unsigned)cur == lo);
    }
    const int wl = __ffs(bal) - 1;
    if (lane == wl) {
      if (MODE != 3) win[j] = cur;
      ++h;
      cur = h < 8 ? nxt : ~0ull;
      nxt = h + 1 < 8 ? (MODE == 2 ? cur + 1 : keys[lane * 8 + h + 1]) : ~0ull;
    }
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
  out[lane] = win[lane] + cur;
}

int main() {
  unsigned long long h[256];
  for (int l = 0; l < 32; ++l)
    for (int i = 0; i < 8; ++i) {
      unsigned v = 0x3f000000u + (unsigned)((l * 7919 + i * 104729) % 100000) * 37u + (unsigned)i * 4000000u;
      h[l * 8 + i] = ((unsigned long long)v << 32) | (unsigned)(l << 16 | i);
    }
  unsigned long long *dk, *dout;
  long long* dc;
  cudaMalloc(&dk, sizeof h);
  cudaMalloc(&dout, 64 * 8);
  cudaMalloc(&dc, 8 * 8);
  cudaMemcpy(dk, h, sizeof h, cudaMemcpyHostToDevice);
  const char* names[] = {"redux", "shfl-min", "redux, no LDS", "redux, no STS"};
  for (int rounds : {1, 8, 32, 64}) {
    for (int m = 0; m < 4; ++m) {
      long long c = 0;
      for (int rep = 0; rep < 3; ++rep) {
        if (m == 0) tourn<0><<<1, 32>>>(dk, dout, dc, rounds);
        if (m == 1) tourn<1><<<1, 32>>>(dk, dout, dc, rounds);
        if (m == 2) tourn<2><<<1, 32>>>(dk, dout, dc, rounds);
        if (m == 3) tourn<3><<<1, 32>>>(dk, dout, dc, rounds);
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      }
      printf("rounds %2d  %-16s %6lld cycles  (%.1f / round)\n", rounds, names[m], c, (double)c / rounds);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
