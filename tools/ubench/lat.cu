// Dependent-chain latencies of the warp-level operations the selection / merge code is built
// from (one warp, or 8 warps for bar.sync), in SM cycles (clock64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench/lat.cu -o /tmp/lat
#include <cstdio>

constexpr int N = 256;

template <int OP>
__global__ void chain(unsigned* out, long long* cyc, unsigned seed) {
  __shared__ unsigned sm[1024];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) & 1023;
  __syncthreads();
  unsigned v = seed + lane;
  double d = (double)v;
  float f = (float)v;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    if (OP == 0) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1u;
    if (OP == 1) v = __reduce_min_sync(0xffffffffu, v) + lane;
    if (OP == 2) v = __ballot_sync(0xffffffffu, v & 1u) + lane;
    if (OP == 3) v = sm[v & 1023];
    if (OP == 4) { asm volatile("bar.sync 1, 256;" ::: "memory"); v += 1; }
    if (OP == 5) f = f * 1.0001f + 1.0f;
    if (OP == 6) d = d * 1.0001 + 1.0;
    if (OP == 7) v = __match_any_sync(0xffffffffu, v & 3u) + lane;
    if (OP == 8) v = (unsigned)__shfl_sync(0xffffffffu, (int)v, v & 31) + 1u;
    if (OP == 9) { unsigned r; asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=r"(r) : "f"(__uint_as_float(v))); v = r + lane; }
    if (OP == 10) v = __popc(__ballot_sync(0xffffffffu, v & 1u)) + v;
    if (OP == 11) { __syncwarp(); v += 1; }
    if (OP == 12) v = (unsigned)__shfl_up_sync(0xffffffffu, (int)v, 1) + 1u;
    if (OP == 13) d = __shfl_xor_sync(0xffffffffu, d, 1) + 1.0;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = v + (unsigned)f + (unsigned)d;
}

template <int OP>
void run(const char* name, int threads) {
  unsigned* o;
  long long* c;
  cudaMalloc(&o, 4096);
  cudaMalloc(&c, 8);
  long long h = 0;
  for (int rep = 0; rep < 3; ++rep) {
    chain<OP><<<1, threads>>>(o, c, 5u);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  }
  printf("%-28s %6.1f cycles per dependent step\n", name, (double)h / N);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<0>("shfl.bfly u32 + iadd", 32);
  run<12>("shfl.up u32 + iadd", 32);
  run<8>("shfl.idx (var src) + iadd", 32);
  run<13>("shfl.bfly f64 + dadd", 32);
  run<1>("redux.min u32 + iadd", 32);
  run<9>("redux.max f32 + iadd", 32);
  run<2>("vote.ballot + iadd", 32);
  run<10>("ballot + popc + iadd", 32);
  run<7>("match.any + iadd", 32);
  run<3>("lds (pointer chase)", 32);
  run<11>("syncwarp + iadd", 32);
  run<4>("bar.sync 8 warps", 256);
  run<5>("ffma", 32);
  run<6>("dfma", 32);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
