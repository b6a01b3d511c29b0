// Consumer-loop microbenchmark for A1 (expand_core.cuh): the streaming CTA of the step kernel
// (producer lane + 8 consumer warps, 5-stage TMA ring of 16 KiB chunks) without the control flow.
//   mode 0 (throughput): every CTA streams `rows_per_cta` whole rows (t = 1, the HBM regime of
//                        cfg5's first layer); reports GB/s over the whole grid.
//   mode 1 (latency):    every CTA streams `nch` chunks of one row (the cfg3 layers' slices);
//                        reports the median time from the first chunk's arrival to the slice end.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//          -I paper_2604_09731_b200/csrc tools/ubench/consume.cu -o tools/ubench/consume
#include <algorithm>
#include <cstdio>
#include <vector>

#include "expand_core.cuh"

using namespace smart;

struct __align__(16) Sh {
  ConsShared cs;
  float2 msl[kMaxCpr * kConsumerWarps];
};

__global__ void fill(unsigned short* x, long long n, int V, unsigned seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 0x9e3779b9u + seed;
    float s = 0.f;
    for (int q = 0; q < 4; ++q) {  // ~N(0, 1) from 4 uniforms
      h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
      s += (h >> 8) * (1.f / 16777216.f);
    }
    float v = (s - 2.f) * 1.732f * 2.f;
    const int e = (int)(i % V);
    if (e % 15991 == 7) v += 14.f - (e % 5);  // a few head tokens per row
    const unsigned u = __float_as_uint(v);
    x[i] = (unsigned short)((u + 0x7fff + ((u >> 16) & 1)) >> 16);
  }
}

__global__ void __launch_bounds__(kLayerThreads, 2)
consume_bench(Params P, const char* __restrict__ logits, long long row_bytes, int mode, int rows_per_cta, int nch,
              unsigned long long* t_out, unsigned long long* keys_out) {
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;
  StreamPipe& pipe = *reinterpret_cast<StreamPipe*>(dsm + kStages * kChunkBytes);
  Sh& sh = *reinterpret_cast<Sh*>(dsm + kStages * kChunkBytes + sizeof(StreamPipe));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    mbar_fence_init();
    sh.cs.tau = 0ull;
  }
  __syncthreads();
  const int cpr = P.cpr, k = P.k;
  const int nrows = mode == 0 ? rows_per_cta : 1;
  const int c0 = mode == 0 ? 0 : (int)(blockIdx.x % (cpr - nch + 1));
  const int c1 = mode == 0 ? cpr : c0 + nch;
  const long long row0 = mode == 0 ? (long long)blockIdx.x * rows_per_cta : blockIdx.x;
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      int i = 0;
      for (int n = 0; n < nrows; ++n) {
        const char* base = logits + (row0 + n) * row_bytes;
        for (int c = c0; c < c1; ++c, ++i) {
          const int st = i % kStages;
          mbar_wait(&pipe.empty[st], ((uint32_t)(i / kStages) & 1u) ^ 1u);
          const long long off = (long long)c * kChunkBytes;
          const uint32_t bytes = (uint32_t)min((long long)kChunkBytes, row_bytes - off);
          mbar_expect_tx(&pipe.full[st], bytes);
          bulk_g2s(ring + (size_t)st * kChunkBytes, base + off, bytes, &pipe.full[st]);
        }
      }
    }
    return;
  }
  unsigned long long tfirst = 0;
  int i = 0, wcnt = 0;
  float wrun = -INFINITY;
  for (int n = 0; n < nrows; ++n) {
    unsigned long long bound = 0ull;
    for (int c = c0; c < c1; ++c, ++i) {
      const int st = i % kStages;
      const char* stage = ring + (size_t)st * kChunkBytes;
      mbar_wait(&pipe.full[st], ((uint32_t)(i / kStages)) & 1u);
      if (i == 0 && tid == 0) tfirst = gtime();
      uint4 raw[kVecPerThread];
      const uint4* sv = reinterpret_cast<const uint4*>(stage);
#pragma unroll
      for (int j = 0; j < kVecPerThread; ++j) raw[j] = sv[j * kConsumers + tid];
      consume_chunk<true, true>(P, sh.cs, sh.msl, raw, stage, nullptr, c, c0, c1, i, wcnt, bound, wrun);
      __syncwarp();
      if (lane == 0) mbar_arrive(&pipe.empty[st]);
    }
    slice_end_post(sh.cs, k, wcnt);
    unsigned long long* gk = keys_out + ((size_t)blockIdx.x * 64 + (n & 63)) * 32;
    slice_end_merge(
#if SMEM_OUT
        sh.cs, sh.msl, k, c1 - c0, [&](int rank, unsigned long long key) { sh.cs.w[0].list[rank & 31] = key; },
        [&](int cc, float M, float S) { sh.cs.w[1].list[cc & 31] = ((unsigned long long)__float_as_uint(M) << 32) | __float_as_uint(S); });
    if (tid == 0) gk[0] = sh.cs.w[0].list[0];
#else
        sh.cs, sh.msl, k, c1 - c0, [&](int rank, unsigned long long key) { gk[rank] = key; },
        [&](int cc, float M, float S) { gk[16 + (cc & 15)] = ((unsigned long long)__float_as_uint(M) << 32) | __float_as_uint(S); });
#endif
    CSTAMP(42);
    consumer_sync();
    CSTAMP(43);
    if (tid == 0) sh.cs.tau = 0ull;
  }
  if (tid == 0) {
    t_out[2 * blockIdx.x] = tfirst;
    t_out[2 * blockIdx.x + 1] = gtime();
  }
}

int main(int argc, char** argv) {
  const int V = argc > 1 ? atoi(argv[1]) : 152064;
  const int k = argc > 2 ? atoi(argv[2]) : 8;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int G = 2 * nsm;
  Params P{};
  P.V = V;
  P.k = k;
  P.chunk_elems = kChunkBytes / 2;
  P.cpr = (V + P.chunk_elems - 1) / P.chunk_elems;
  const long long row_bytes = (long long)V * 2;
  const int rows_per_cta = 4;
  const long long nrows_pool = (long long)G * rows_per_cta;
  const int npool = 4;  // rotating pools: > 2x L2
  unsigned short* x = nullptr;
  cudaMalloc(&x, nrows_pool * row_bytes * npool);
  fill<<<1024, 256>>>(x, nrows_pool * V * npool, V, 12345u);
  unsigned long long *t = nullptr, *keys = nullptr;
  cudaMalloc(&t, G * 16);
  cudaMalloc(&keys, (size_t)G * 64 * 32 * 8);
  const size_t smem = kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(Sh);
  cudaFuncSetAttribute(consume_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // mode 0: throughput
  for (int rep = 0; rep < 3; ++rep)
    consume_bench<<<G, kLayerThreads, smem>>>(P, (const char*)x + rep % npool * nrows_pool * row_bytes, row_bytes, 0,
                                               rows_per_cta, 0, t, keys);
  std::vector<float> ms;
  for (int rep = 0; rep < 12; ++rep) {
    cudaEventRecord(e0);
    consume_bench<<<G, kLayerThreads, smem>>>(P, (const char*)x + rep % npool * nrows_pool * row_bytes, row_bytes, 0,
                                               rows_per_cta, 0, t, keys);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float m = 0;
    cudaEventElapsedTime(&m, e0, e1);
    ms.push_back(m);
  }
  std::sort(ms.begin(), ms.end());
  const double bytes = (double)nrows_pool * row_bytes;
#if CONSUME_COUNTS
  {
    unsigned long long cnt[8];
    cudaMemcpyFromSymbol(cnt, g_ccount, sizeof cnt);
    printf("counts over 15 launches: warp-chunks %llu, with candidates %llu, candidates %llu, expansion passes %llu, "
           "mid-chunk compactions %llu, end-of-chunk compactions %llu\n", cnt[0], cnt[1], cnt[2], cnt[5], cnt[3], cnt[4]);
  }
#endif
  printf("V %d k %d: throughput mode, %d CTAs x %d rows: %.1f MB in %.2f us (median) = %.0f GB/s  [err %s]\n", V, k, G,
         rows_per_cta, bytes / 1e6, ms[ms.size() / 2] * 1e3, bytes / (ms[ms.size() / 2] * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  // mode 1: latency of 1- and 2-chunk slices
  for (int nch = 1; nch <= 3; ++nch) {
    std::vector<double> lat;
    for (int rep = 0; rep < 8; ++rep) {
      consume_bench<<<G, kLayerThreads, smem>>>(P, (const char*)x + (rep % npool) * nrows_pool * row_bytes, row_bytes, 1,
                                                 1, nch, t, keys);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> h(2 * G);
      cudaMemcpy(h.data(), t, 16 * G, cudaMemcpyDeviceToHost);
      for (int b = 0; b < G; ++b) lat.push_back((h[2 * b + 1] - h[2 * b]) / 1e3);
    }
#if CONSUME_STAMPS
    unsigned long long st[64];
    cudaMemcpyFromSymbol(st, g_cstamp, sizeof st);
    printf("  CTA0 warp0 cycles from chunk start:");
    for (int q = 0; q < 8 * nch; ++q) printf(" %lld", (long long)(st[q] - st[0]));
    printf(" | post %lld synced %lld merged %lld end %lld\n", (long long)(st[40] - st[0]), (long long)(st[41] - st[0]),
           (long long)(st[42] - st[0]), (long long)(st[43] - st[0]));
#endif
    std::sort(lat.begin(), lat.end());
    printf("latency mode, %d chunk(s) per CTA, %d CTAs: first-chunk arrival -> slice end median %.2f us, p90 %.2f us\n",
           nch, G, lat[lat.size() / 2], lat[lat.size() * 9 / 10]);
  }
  return 0;
}
