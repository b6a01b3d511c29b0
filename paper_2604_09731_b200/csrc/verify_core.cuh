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

// One 16 KiB chunk (base element cbase) of a verify row, by one consumer warp: exact argmax of the
// chunk (value desc, index asc) folded into the segment's running best (bv, bi); vector maxima on
// packed values (bf16x2 max), one-instruction warp max, then the index is searched only in the
// vectors holding it.  SAMPLE (T > 0): the same on the perturbed logits x / tau + G (recomputed
// bit-identically for the index search).  A NaN logit sets nanf (Q23).
template <bool BF16, bool SAMPLE>
__device__ __forceinline__ void verify_chunk(uint4 (&raw)[kVecPerThread], int cbase, int V, int tid, uint32_t rowkey,
                                             float inv_tau, float& bv, int& bi, int& nanf) {
  constexpr int EPV = BF16 ? 8 : 4;
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
