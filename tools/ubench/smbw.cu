// per-SM TMA streaming bandwidth (debug aid): G CTAs each stream `bytes` contiguous bytes with a
// kS-stage ring of 16 KiB bulk copies; consumers touch one word per 16 B (sum) to keep it honest.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kChunk = 16384;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int S>
__global__ void __launch_bounds__(288) stream(const char* src, long long bytes, unsigned long long* out, float* sink) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * kChunk);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + (long long)blockIdx.x * bytes;
  const int n = (int)(bytes / kChunk);
  unsigned long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (warp == 8) {
    if (lane == 0)
      for (int i = 0; i < n; ++i) {
        const int s = i % S;
        const uint32_t ph = ((i / S) & 1) ^ 1;
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(su(&empty[s])), "r"(ph) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(kChunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + s * kChunk)), "l"(base + (long long)i * kChunk), "r"(kChunk), "r"(su(&full[s])) : "memory");
      }
    return;
  }
  float acc = 0.f;
  for (int i = 0; i < n; ++i) {
    const int s = i % S;
    const uint32_t ph = (i / S) & 1;
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(su(&full[s])), "r"(ph) : "memory");
    const uint4* st = reinterpret_cast<const uint4*>(sm + s * kChunk);
#pragma unroll
    for (int j = 0; j < 4; ++j) { uint4 v = st[j * 256 + tid]; acc += __uint_as_float(v.x) + __uint_as_float(v.w); }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
  }
  asm volatile("bar.sync 1, 256;");
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (tid == 0) { out[blockIdx.x] = t1 - t0; sink[blockIdx.x] = acc; }
}
template <int S>
void run(int G, long long bytes, const char* src, unsigned long long* out, float* sink) {
  size_t smem = S * kChunk + 2 * S * 8;
  cudaFuncSetAttribute(stream<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) stream<S><<<G, 288, smem>>>(src, bytes, out, sink);
  cudaEventRecord(e0);
  const int R = 10;
  const long long span = (long long)G * bytes; const int nrot = (int)((1ll << 30) / span);
  for (int rep = 0; rep < R; ++rep) stream<S><<<G, 288, smem>>>(src + (nrot > 1 ? (rep % nrot) * span : 0), bytes, out, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2048]; cudaMemcpy(h, out, G * 8, cudaMemcpyDeviceToHost);
  double mx = 0, mn = 1e30; for (int b = 0; b < G; ++b) { mx = h[b] > mx ? h[b] : mx; mn = h[b] < mn ? h[b] : mn; }
  printf("S=%2d G=%4d bytes/CTA=%7lld KB: kernel %.2f us (launch-incl), in-kernel CTA time min %.2f max %.2f us, per-CTA GB/s %.1f, total GB/s %.0f\n",
         S, G, bytes / 1024, ms * 1000 / R, mn / 1000, mx / 1000, bytes / (mx / 1e9) / 1e9, (double)G * bytes / (ms / R / 1e3) / 1e9);
}
int main() {
  const long long maxb = 1ll << 30;
  char* src; cudaMalloc(&src, maxb);
  cudaMemset(src, 0, maxb);
  unsigned long long* out; cudaMalloc(&out, 4096 * 8);
  float* sink; cudaMalloc(&sink, 4096 * 4);
  for (long long kb : {304, 1216}) {
    for (int G : {148, 256, 296, 444}) {
      if ((long long)G * kb * 1024 > maxb) continue;
      run<4>(G, kb * 1024, src, out, sink);
      run<5>(G, kb * 1024, src, out, sink);
      run<8>(G, kb * 1024, src, out, sink);
    }
  }
  return 0;
}
