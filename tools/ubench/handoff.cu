// Cross-CTA handoff latency (debug aid for the step kernel's slice-end -> selection path):
// S producer CTAs each write a small record (8 keys + 2 partials, like a slice list) and signal;
// one consumer CTA waits for all S and reads the records.  Per round: the consumer releases a
// "go" word, producers see it, write, signal; latency = consumer done - latest producer signal.
//   V0: bar.sync + red.release.gpu counter; consumer: relaxed poll + fence.acq_rel, ld.cg records
//   V1: self-validating records: 16-byte words {data, tag} written with st.relaxed.v2; the
//       consumer polls each word until its tag matches (no counter, no fence)
//   V2: V0 without any fence (red.relaxed; consumer relaxed poll, no fence): the fence cost only
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench/handoff.cu -o /tmp/handoff
#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ld_relaxed_v2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_v2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

constexpr int kWords = 10;  // 16-byte words per record (V1) / 8-byte words (V0, V2)

template <int VAR>
__global__ void handoff(int S, int rounds, int* go, int* arrive, unsigned long long* rec, unsigned long long* tsig,
                        unsigned long long* tdone, unsigned long long* sink) {
  const int tid = threadIdx.x;
  __shared__ int s_round;
  if (blockIdx.x == 0) {  // consumer
    unsigned long long acc = 0;
    for (int r = 1; r <= rounds; ++r) {
      __syncthreads();
      if (tid == 0) {
        asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(go), "r"(r) : "memory");
      }
      if (VAR == 1) {
        for (int e = tid; e < S * kWords; e += blockDim.x) {
          unsigned long long a, b;
          do {
            ld_relaxed_v2(rec + 2 * (size_t)e, a, b);
          } while (b != (unsigned long long)r);
          acc += a;
        }
      } else {
        if (tid == 0) {
          while (ld_relaxed(arrive) < S * r) {
          }
          if (VAR == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        for (int e = tid; e < S * kWords; e += blockDim.x) acc += __ldcg(rec + e);
      }
      __syncthreads();
      if (tid == 0) tdone[r] = gtime();
    }
    sink[tid] = acc;
  } else {  // producer s
    const int s = blockIdx.x - 1;
    for (int r = 1; r <= rounds; ++r) {
      if (tid == 0) {
        while (ld_relaxed(go) < r) {
        }
        s_round = r;
      }
      __syncthreads();
      if (VAR == 1) {
        if (tid < kWords) st_relaxed_v2(rec + 2 * ((size_t)s * kWords + tid), (unsigned long long)(s * 100 + tid), r);
        if (tid == 0) tsig[(size_t)r * S + s] = gtime();
      } else {
        if (tid < kWords) rec[(size_t)s * kWords + tid] = (unsigned long long)(s * 100 + tid + r);
        __syncthreads();
        if (tid == 0) {
          tsig[(size_t)r * S + s] = gtime();
          if (VAR == 0)
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(arrive) : "memory");
          else
            asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(arrive) : "memory");
        }
      }
      __syncthreads();
    }
  }
}

int main() {
  const int rounds = 200;
  for (int S : {16, 64, 256}) {
    for (int var = 0; var < 3; ++var) {
      int *go, *arrive;
      unsigned long long *rec, *tsig, *tdone, *sink;
      cudaMalloc(&go, 4);
      cudaMalloc(&arrive, 4);
      cudaMalloc(&rec, (size_t)S * kWords * 16);
      cudaMalloc(&tsig, (size_t)(rounds + 1) * S * 8);
      cudaMalloc(&tdone, (size_t)(rounds + 1) * 8);
      cudaMalloc(&sink, 1024 * 8);
      cudaMemset(go, 0, 4);
      cudaMemset(arrive, 0, 4);
      cudaMemset(rec, 0, (size_t)S * kWords * 16);
      if (var == 0) handoff<0><<<S + 1, 256>>>(S, rounds, go, arrive, rec, tsig, tdone, sink);
      if (var == 1) handoff<1><<<S + 1, 256>>>(S, rounds, go, arrive, rec, tsig, tdone, sink);
      if (var == 2) handoff<2><<<S + 1, 256>>>(S, rounds, go, arrive, rec, tsig, tdone, sink);
      cudaError_t err = cudaDeviceSynchronize();
      std::vector<unsigned long long> hs((size_t)(rounds + 1) * S), hd(rounds + 1);
      cudaMemcpy(hs.data(), tsig, hs.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hd.data(), tdone, hd.size() * 8, cudaMemcpyDeviceToHost);
      std::vector<double> lat;
      for (int r = 10; r <= rounds; ++r) {
        unsigned long long mx = 0;
        for (int s = 0; s < S; ++s) mx = std::max(mx, hs[(size_t)r * S + s]);
        lat.push_back((double)(long long)(hd[r] - mx));
      }
      std::sort(lat.begin(), lat.end());
      printf("S %3d V%d (%s): latest signal -> consumer done: median %.0f ns, p10 %.0f, p90 %.0f [%s]\n", S, var,
             var == 0 ? "counter + release/acquire" : var == 1 ? "tagged 16-byte records" : "counter, no fences",
             lat[lat.size() / 2], lat[lat.size() / 10], lat[lat.size() * 9 / 10], cudaGetErrorString(err));
      cudaFree(go);
      cudaFree(arrive);
      cudaFree(rec);
      cudaFree(tsig);
      cudaFree(tdone);
      cudaFree(sink);
    }
  }
  return 0;
}
