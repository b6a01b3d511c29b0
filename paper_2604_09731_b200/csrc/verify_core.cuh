// verify_core.cuh — the per-chunk work of A8 (target argmax of a tree row, P:453 T = 0)
// and of its T > 0 variant (NEXT #1, Gumbel-max sample, Q31), shared by the verify kernel
// (mask_verify.cu) and the persistent whole-step kernel (step.cu).
#pragma once

#include "stream.cuh"

namespace smart {

__device__ __forceinline__ uint32_t bmax2_nan(uint32_t a, uint32_t b) {  // packed bf16x2 max, NaN-propagating
  uint32_t d;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t vkey_orderable(float f) {  // order-preserving float -> u32
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}


// NEXT #1 (Q31): perturbed logit of token v at a verify row: x / tau + Gumbel(U_v), with
// U_v = ((h >> 9) + 1/2) / 2^23, h = lowbias32(rowkey + v * 0x9e3779b9) and rowkey the high
// half of SplitMix64(seed + (global request << 22 | node) * golden-gamma), computed once per
// row.  U is exact in fp32; G is evaluated in fp32 (the oracle in fp64), decisions closer than
// 1e-4 are tie-ambiguous (Q24).
__device__ __forceinline__ uint32_t sample_rowkey(unsigned long long seed, unsigned long long r, unsigned long long node) {
  unsigned long long z = seed + ((r << 22) | node) * 0x9e3779b97f4a7c15ull;
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return (uint32_t)(z >> 32);
}
__device__ __forceinline__ float perturbed(float x, float inv_tau, uint32_t rowkey, int v) {
  uint32_t h = rowkey + (uint32_t)v * 0x9e3779b9u;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  const float U = ((float)(h >> 9) + 0.5f) * 1.1920928955078125e-07f;
  // -ln U: series in t = 1 - U (exact) near U = 1, fast log elsewhere (|error| in G < 3e-5)
  const float t = 1.0f - U;
  const float e = (t < 0.015625f) ? t * (1.0f + t * (0.5f + t * (0.33333334f + t * 0.25f))) : -__logf(U);
  return fmaf(x, inv_tau, -__logf(e));
}

// T > 0 (Q31) with pruning: G = -ln(-ln U) <= 16.64 for every 23-bit U, and G <= 6.92 unless
// U >= 0.999 (the computed G is within 3e-5 of the exact one), so a token can reach the bound T (a
// perturbed value some token of the row attains) only if fma(x, 1/tau, Gmax(U)) >= T; the 23-bit
// hash decides which Gmax applies, and the two logarithms are evaluated only for the tokens that
// pass.  T = max(running best of the segment, exact perturbed value of the warp's largest x).
// Exact: the winning token passes its own test (the rounding of fma is monotone in the addend).
constexpr uint32_t kU999 = 8380000u;  // (h >> 9) >= this  <=>  U >= ~0.99898
// the hash before its last xor-shift: that step keeps bits 31..16, so h >= kU999 << 9 = 0xFFBCC000
// implies (h before it) >= 0xFFBC0000; testing the latter marks a superset of the large-G tokens
// (the bound stays valid) and saves the last two operations of the per-token hash
constexpr uint32_t kU999Pre = 0xFFBC0000u;
static_assert((kU999 << 9) == 0xFFBCC000u, "kU999Pre follows kU999");
__device__ __forceinline__ uint32_t sample_hash_pre(uint32_t rowkey, int v) {
  uint32_t h = rowkey + (uint32_t)v * 0x9e3779b9u;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  return h;
}
template <bool BF16>
__device__ __forceinline__ void sample_chunk(const uint4 (&raw)[kVecPerThread], int cbase, int V, int tid, uint32_t rowkey,
                                             float inv_tau, float& bv, int& bi, int& nanf) {
  constexpr int EPV = BF16 ? 8 : 4;
  constexpr int EPT = kVecPerThread * EPV;  // 32 elements per thread
  auto xat = [&](const uint4& q, int e) {
    const int wi = BF16 ? e >> 1 : e;
    const uint32_t w = wi == 0 ? q.x : wi == 1 ? q.y : wi == 2 ? q.z : q.w;
    return BF16 ? __uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16)) : __uint_as_float(w);
  };
  const bool ragged = cbase + kChunkBytes / (BF16 ? 2 : 4) > V;
  // (1) the warp's largest logit x* (packed maxima, NaN-propagating) and its exact perturbed value
  float vm[kVecPerThread];
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    if (BF16) {
      const uint32_t mw = bmax2_nan(bmax2_nan(raw[j].x, raw[j].y), bmax2_nan(raw[j].z, raw[j].w));
      vm[j] = fmax_nan(__uint_as_float(mw << 16), __uint_as_float(mw & 0xffff0000u));
    } else {
      vm[j] = fmax_nan(fmax_nan(__uint_as_float(raw[j].x), __uint_as_float(raw[j].y)),
                       fmax_nan(__uint_as_float(raw[j].z), __uint_as_float(raw[j].w)));
    }
    if (ragged) {  // elements past the row end never take part: the vector maximum over the rest
      const int e0 = cbase + (j * kConsumers + tid) * EPV;
      if (e0 + EPV > V) {
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < EPV; ++e)
          if (e0 + e < V) mx = fmax_nan(mx, xat(raw[j], e));
        vm[j] = mx;
      }
    }
  }
  float m = fmax_nan(fmax_nan(vm[0], vm[1]), fmax_nan(vm[2], vm[3]));
  if (m != m) {  // a NaN logit: flagged (Q23); the row's sample is then unspecified
    nanf = 1;
    m = -INFINITY;
  }
  // the bound: every lane's own largest element, perturbed exactly; T = the warp's maximum
  float ps = -INFINITY;
  if (m != -INFINITY) {
    int jb = 0;
#pragma unroll
    for (int j = kVecPerThread - 1; j >= 0; --j) jb = vm[j] == m ? j : jb;  // first vector holding m
    uint4 q = raw[0];
#pragma unroll
    for (int j = 1; j < kVecPerThread; ++j) q = jb == j ? raw[j] : q;
    const int e0 = cbase + (jb * kConsumers + tid) * EPV;
    int eb = 0;
#pragma unroll
    for (int e = EPV - 1; e >= 0; --e) eb = (xat(q, e) == m && e0 + e < V) ? e : eb;
    ps = perturbed(m, inv_tau, rowkey, e0 + eb);
  }
  ps = warp_max_fast(ps);
  const float T = fmaxf(bv, ps);
  // (2) candidate mask, branch-free: fma(x, 1/tau, Gmax(U)) >= T
  uint32_t cm = 0u;
#pragma unroll
  for (int n = 0; n < EPT; ++n) {
    const int j = n / EPV, e = n % EPV;
    const int v = cbase + (j * kConsumers + tid) * EPV + e;
    const uint32_t h = sample_hash_pre(rowkey, v);
    const float gmax = h >= kU999Pre ? 16.64f : 6.92f;
    cm |= (fmaf(xat(raw[j], e), inv_tau, gmax) >= T && (!ragged || v < V)) ? (1u << n) : 0u;
  }
  // (3) exact perturbed values of the candidates only (rare), the lane's best, the warp's
  float pv = -INFINITY;
  int pi = kIdxSentinel;
  while (cm) {
    const int n = __ffs(cm) - 1;
    cm &= cm - 1u;
    const int j = n / EPV, e = n % EPV;
    const int v = cbase + (j * kConsumers + tid) * EPV + e;
    const uint4 q = raw[j];
    const int wi = BF16 ? e >> 1 : e;
    const uint32_t w = wi == 0 ? q.x : wi == 1 ? q.y : wi == 2 ? q.z : q.w;
    const float x = BF16 ? __uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16)) : __uint_as_float(w);
    const float p = perturbed(x, inv_tau, rowkey, v);
    if (p > pv) {  // candidates in increasing index order: ties keep the lower index
      pv = p;
      pi = v;
    }
  }
  const float Mw = warp_max_fast(pv);
  const int mi = (int)__reduce_min_sync(kFull, (unsigned)(pv == Mw ? pi : kIdxSentinel));
  if (mi != kIdxSentinel && better(Mw, mi, bv, bi)) {
    bv = Mw;
    bi = mi;
  }
}

// One 16 KiB chunk (base element cbase) of a verify row, by one consumer warp: exact argmax of the
// chunk (value desc, index asc) folded into the segment's running best (bv, bi); vector maxima on
// packed values (bf16x2 max), one-instruction warp max, then the index is searched only in the
// vectors holding it.  SAMPLE (T > 0): the same on the perturbed logits x / tau + G (recomputed
// bit-identically for the index search).  A NaN logit sets nanf (Q23).
template <bool BF16, bool SAMPLE>
__device__ __forceinline__ void verify_chunk(uint4 (&raw)[kVecPerThread], int cbase, int V, int tid, uint32_t rowkey,
                                             float inv_tau, float& bv, int& bi, int& nanf) {
  constexpr int EPV = BF16 ? 8 : 4;
  if (SAMPLE) {
    sample_chunk<BF16>(raw, cbase, V, tid, rowkey, inv_tau, bv, bi, nanf);
    return;
  }
  if (cbase + kChunkBytes / (BF16 ? 2 : 4) > V) {  // ragged last chunk: elements past the row end -> -inf
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const int e0 = cbase + (j * kConsumers + tid) * EPV;
      uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
      for (int e = 0; e < EPV; ++e)
        if (e0 + e >= V) {
          if (BF16) w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0x0000ffffu) | 0xff800000u) : ((w[e >> 1] & 0xffff0000u) | 0xff80u);
          else w[e] = 0xff800000u;
        }
      raw[j] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  // ---- exact argmax of this (chunk, warp): vector maxima on packed values (bf16x2 max),
  // one-instruction warp max, then the index is searched only in the vectors holding it.
  // SAMPLE (T > 0): the same on the perturbed logits x / tau + G (recomputed bit-identically
  // for the index search) ----
  auto xat = [&](const uint32_t (&w)[4], int e) {
    return BF16 ? __uint_as_float((e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16))
                : __uint_as_float(w[e]);
  };
  float vm[kVecPerThread];
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    if (SAMPLE) {
      const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
      const int e0 = cbase + (j * kConsumers + tid) * EPV;
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < EPV; ++e) mx = fmax_nan(mx, perturbed(xat(w, e), inv_tau, rowkey, e0 + e));
      vm[j] = mx;
    } else if (BF16) {
      const uint32_t mw = bmax2_nan(bmax2_nan(raw[j].x, raw[j].y), bmax2_nan(raw[j].z, raw[j].w));
      vm[j] = fmax_nan(__uint_as_float(mw << 16), __uint_as_float(mw & 0xffff0000u));
    } else {
      vm[j] = fmax_nan(fmax_nan(__uint_as_float(raw[j].x), __uint_as_float(raw[j].y)),
                       fmax_nan(__uint_as_float(raw[j].z), __uint_as_float(raw[j].w)));
    }
  }
  float m = fmax_nan(fmax_nan(vm[0], vm[1]), fmax_nan(vm[2], vm[3]));
  if (m != m) {  // a NaN logit: flagged (Q23); the row's argmax is then unspecified
    nanf = 1;
    m = -INFINITY;
  }
  const float Mw = warp_max_fast(m);
  int li = kIdxSentinel;
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j)
    if (vm[j] == Mw) {
      const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
      const int e0 = cbase + (j * kConsumers + tid) * EPV;
#pragma unroll
      for (int e = 0; e < EPV; ++e) {
        const float xv = SAMPLE ? perturbed(xat(w, e), inv_tau, rowkey, e0 + e) : xat(w, e);
        if (xv == Mw && e0 + e < V) li = min(li, e0 + e);
      }
    }
  const int mi = (int)__reduce_min_sync(kFull, (unsigned)li);
  if (better(Mw, mi, bv, bi)) {
    bv = Mw;
    bi = mi;
  }
}

}  // namespace smart
