// Row-merge microbenchmark (expand_core.cuh merge_row_tournament): one CTA of 8 warps merges R rows
// of t sorted slice lists (k keys each) + cpr chunk partials staged in shared memory, one warp per
// row, rows round-robin; clock64 per warp.  Variants: 0 full merge, 1 Z only, 2 tournament only.
#include <cstdio>
#include <vector>

#include "expand_core.cuh"

using namespace smart;

template <int VAR>
__global__ void merge_bench(const unsigned long long* gkeys, const float2* gms, int R, int t, int k, int cpr,
                            unsigned long long* out, long long* cyc) {
  extern __shared__ __align__(16) char sm[];
  const int kp = list_stride(k);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(sm);
  float2* ms = reinterpret_cast<float2*>(keys + (size_t)R * t * kp);
  for (int e = threadIdx.x; e < R * t * kp; e += blockDim.x) keys[e] = gkeys[e];
  for (int e = threadIdx.x; e < R * cpr; e += blockDim.x) ms[e] = gms[e];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t0 = clock64();
  for (int row = warp; row < R; row += 8) {
    const unsigned long long* kr = keys + (size_t)row * t * kp;
    const float2* mr = ms + (size_t)row * cpr;
    auto msf = [&](int c) {
      const float2 v = mr[c];
      return make_float4(v.x, v.y, 0.f, 0.f);
    };
    if (VAR == 0) {
      merge_row_tournament(k, cpr, t, 0.5f, msf, kr,
                           [&](int rank, int tok, float p, float cum) {
                             out[row * 32 + rank] = ((unsigned long long)tok << 32) | __float_as_uint(cum);
                           });
    } else if (VAR == 1) {
      const float4 v0 = lane < cpr ? msf(lane) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
      const float M = warp_max_fast(v0.x);
      const float z = v0.y * ex2(fmaf(v0.x, kLog2e, -M * kLog2e));
      const float Z = warp_sum(z);
      if (lane == 0) out[row * 32] = __float_as_uint(__frcp_rn(Z));
    } else if (VAR == 3 || VAR == 4) {
      // branch-free: every lane reloads its (possibly advanced) next entry each round from a
      // 32-bit shared address; VAR 4 interleaves two rows per warp
      constexpr int NR = VAR == 4 ? 2 : 1;
      unsigned long long cur[NR], nxt[NR], mine[NR];
      int h[NR];
      uint32_t base[NR];
      bool own = lane < t;
      for (int q = 0; q < NR; ++q) {
        const int rr = min(row + q * 8, R - 1);
        base[q] = smem_u32(keys + (size_t)rr * t * kp + lane * kp);
        cur[q] = own ? keys[(size_t)rr * t * kp + lane * kp] : 0ull;
        nxt[q] = own ? keys[(size_t)rr * t * kp + lane * kp + 1] : 0ull;
        h[q] = 1;
        mine[q] = 0;
      }
      for (int r = 0; r < k; ++r) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const unsigned hi = __reduce_max_sync(kFull, (unsigned)(cur[q] >> 32));
          const unsigned lo = __reduce_max_sync(kFull, (unsigned)(cur[q] >> 32) == hi ? (unsigned)cur[q] : 0u);
          const unsigned long long win = ((unsigned long long)hi << 32) | lo;
          mine[q] = lane == r ? win : mine[q];
          const bool adv = own && cur[q] == win;
          cur[q] = adv ? nxt[q] : cur[q];
          h[q] += adv ? 1 : 0;
          unsigned long long ld;
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ld) : "r"(base[q] + 8u * (uint32_t)min(h[q], k - 1)));
          nxt[q] = adv ? (h[q] < k ? ld : 0ull) : nxt[q];
        }
      }
      for (int q = 0; q < NR; ++q)
        if (lane < k && row + q * 8 < R) out[(row + q * 8) * 32 + lane] = mine[q];
      if (VAR == 4) row += 8;
    } else if (VAR == 7) {
      unsigned long long* sv = reinterpret_cast<unsigned long long*>(ms + (size_t)R * cpr) + warp * 32 * 9;
      merge_row_rank(k, cpr, t, 0.5f, msf, kr, sv, [&](int rank, int tok, float p, float cum) {
        out[row * 32 + rank] = ((unsigned long long)tok << 32) | __float_as_uint(cum);
      });
    } else if (VAR == 6) {
      // tournament with a 5-step shuffle butterfly on the 64-bit key (no redux)
      const bool own = lane < t;
      const uint32_t base = smem_u32(keys + (size_t)row * t * kp + lane * kp);
      unsigned long long cur = own ? kr[lane * kp] : 0ull, nxt = own ? kr[lane * kp + 1] : 0ull, mine = 0;
      int h = 1;
      for (int r = 0; r < k; ++r) {
        unsigned long long w = cur;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long u = __shfl_xor_sync(kFull, w, o);
          w = u > w ? u : w;
        }
        mine = lane == r ? w : mine;
        const bool adv = own && cur == w;
        cur = adv ? nxt : cur;
        h += adv ? 1 : 0;
        unsigned long long ld;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ld) : "r"(base + 8u * (uint32_t)min(h, k - 1)));
        nxt = adv ? (h < k ? ld : 0ull) : nxt;
      }
      if (lane < k) out[row * 32 + lane] = mine;
    } else if (VAR == 5) {
      // one REDUX per round: the value word's max; its holders by ballot; the index word's max only
      // on a value tie (rare); the winner lane stores its key at slot r and advances
      const bool own = lane < t;
      const uint32_t base = smem_u32(keys + (size_t)row * t * kp + lane * kp);
      unsigned long long* res = reinterpret_cast<unsigned long long*>(ms + (size_t)R * cpr) + warp * 32;
      unsigned long long cur = own ? kr[lane * kp] : 0ull, nxt = own ? kr[lane * kp + 1] : 0ull;
      int h = 1;
      for (int r = 0; r < k; ++r) {
        const unsigned chi = (unsigned)(cur >> 32);
        const unsigned hi = __reduce_max_sync(kFull, chi);
        bool win = own && chi == hi;
        const unsigned bal = __ballot_sync(kFull, win);
        if (bal & (bal - 1u)) {  // value tie: the larger index word (lower token id) wins
          const unsigned lo = __reduce_max_sync(kFull, win ? (unsigned)cur : 0u);
          win = win && (unsigned)cur == lo;
        }
        if (win) res[r] = cur;
        cur = win ? nxt : cur;
        h += win ? 1 : 0;
        unsigned long long ld;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ld) : "r"(base + 8u * (uint32_t)min(h, k - 1)));
        nxt = win ? (h < k ? ld : 0ull) : nxt;
      }
      __syncwarp();
      if (lane < k) out[row * 32 + lane] = res[lane];
    } else {
      const bool own = lane < t;
      unsigned long long cur = own ? kr[lane * kp] : 0ull, nxt = own ? kr[lane * kp + 1] : 0ull, mine = 0;
      int h = 1;
      for (int r = 0; r < k; ++r) {
        const unsigned hi = __reduce_max_sync(kFull, (unsigned)(cur >> 32));
        const unsigned lo = __reduce_max_sync(kFull, (unsigned)(cur >> 32) == hi ? (unsigned)cur : 0u);
        const unsigned long long win = ((unsigned long long)hi << 32) | lo;
        if (lane == r) mine = win;
        if (own && cur == win) {
          cur = nxt;
          ++h;
          nxt = h < k ? kr[lane * kp + h] : 0ull;
        }
      }
      if (lane < k) out[row * 32 + lane] = mine;
    }
  }
  __syncwarp();
  const long long t1 = clock64();
  if (lane == 0) cyc[warp] = t1 - t0;
}

int main() {
  const int R = 32, t = 9, k = 8, cpr = 16, kp = 8;
  std::vector<unsigned long long> hk((size_t)R * t * kp);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s; };
  for (int r = 0; r < R; ++r)
    for (int m = 0; m < t; ++m) {
      unsigned v = 0xC0000000u + (rnd() >> 8);
      for (int j = 0; j < kp; ++j) {
        v -= rnd() >> 16;
        hk[((size_t)r * t + m) * kp + j] = ((unsigned long long)v << 32) | (0xffffffffu - (m * 1000 + j));
      }
    }
  std::vector<float2> hm((size_t)R * cpr);
  for (auto& x : hm) x = make_float2((rnd() >> 20) * 1e-3f, 100.f + (rnd() >> 24));
  unsigned long long *dk, *dout;
  float2* dm;
  long long* dc;
  cudaMalloc(&dk, hk.size() * 8);
  cudaMalloc(&dm, hm.size() * 8);
  cudaMalloc(&dout, R * 32 * 8);
  cudaMalloc(&dc, 8 * 8);
  cudaMemcpy(dk, hk.data(), hk.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dm, hm.data(), hm.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = hk.size() * 8 + hm.size() * 8 + 8 * 32 * 9 * 8;
  for (int var = 0; var < 16; ++var) {
    const int thr = var >= 8 ? 32 : 256;
    for (int rep = 0; rep < 3; ++rep) {
      if (var % 8 == 0) merge_bench<0><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 1) merge_bench<1><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 2) merge_bench<2><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 3) merge_bench<3><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 4) merge_bench<4><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 5) merge_bench<5><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 6) merge_bench<6><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
      if (var % 8 == 7) merge_bench<7><<<1, thr, smem>>>(dk, dm, R, t, k, cpr, dout, dc);
    }
    if (var % 8 == 4 || var % 8 == 5 || var % 8 == 6) continue;
    long long c[8];
    cudaMemcpy(c, dc, 64, cudaMemcpyDeviceToHost);
    const int v = var % 8;
    const int rows_per_warp = R / 8;
    printf("variant %d (%s) %s: cycles warp0 %lld -> %.0f cycles/row  [%s]\n", v,
           v == 0 ? "full" : v == 1 ? "Z only" : v == 2 ? "tournament" : v == 3 ? "branch-free" : v == 4 ? "x2 rows" : v == 5 ? "1 REDUX/round" : v == 6 ? "shfl butterfly" : "threshold+rank",
           thr == 32 ? "1 warp " : "8 warps", c[0], c[0] / (double)rows_per_warp, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
