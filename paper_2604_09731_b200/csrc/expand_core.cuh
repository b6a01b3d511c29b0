// expand_core.cuh — the consumer side of A1 (top-k + softmax partials of a streamed logit row,
// P:216-222), shared by the per-layer kernel (expand.cu) and the persistent whole-step
// kernel (step.cu).
//
// A CTA's 8 consumer warps take a slice [mlo, mhi) of one row's 16 KiB chunks from the TMA ring:
//  * softmax: per (chunk, warp) a fixed-tree partial (max, sum exp) — FFMA2 + MUFU.EX2 + FADD2 on
//    element pairs, xor-tree sum; per chunk the 8 warp partials are combined in warp order at the
//    slice end, and the row's cpr chunk partials in lane-strided order by the row merge, so Z is
//    bit-identical for any team layout or sharding.
//  * top-k (exact, ties -> lower index, Q9): 64-bit keys (orderable value | ~index); per warp a
//    running lower bound of the slice's k-th best key (first chunk: the k-th largest of the 8
//    warps' top-j lane maxima; later: compactions and a barrier-free CTA hint, sh.tau); only
//    16-byte vectors whose max reaches the bound are expanded (cooperatively, 8 lanes per vector)
//    and appended to the warp buffer, compacted to its top-k by rank counting when full.
//  * slice end: the CTA's top-k by a rank merge of the 8 padded warp lists, and the per-chunk
//    (M_c, S_c) pairs.
#pragma once

#include "stream.cuh"

namespace smart {

#ifndef CONSUME_STAMPS
#define CONSUME_STAMPS 0  // tools/ubench/consume.cu only: clock64 stamps of CTA 0, warp 0
#endif
#ifndef CONSUME_COUNTS
#define CONSUME_COUNTS 0  // tools/ubench/consume.cu only: slow-path counters
#endif
#if CONSUME_COUNTS
__device__ unsigned long long g_ccount[8];
#define CCOUNT(i, v) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_ccount[i], (unsigned long long)(v))
#else
#define CCOUNT(i, v)
#endif
#if CONSUME_STAMPS
__device__ unsigned long long g_cstamp[64];
#define CSTAMP(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_cstamp[i] = clock64()
#else
#define CSTAMP(i)
#endif

template <bool BF16>
struct Traits {
  static constexpr int EPV = BF16 ? 8 : 4;         // elements per 16 B vector
  static constexpr int EPT = kVecPerThread * EPV;  // elements per consumer thread per chunk
};

// element n (= j*EPV + e) of consumer thread `tid` in a chunk -> row element index
template <bool BF16>
__device__ __forceinline__ int elem_index(int chunk_base, int tid, int n) {
  constexpr int EPV = Traits<BF16>::EPV;
  return chunk_base + ((n / EPV) * kConsumers + tid) * EPV + (n % EPV);
}

template <bool BF16>
__device__ __forceinline__ void unpack(const uint4 (&raw)[kVecPerThread], float (&x)[Traits<BF16>::EPT]) {
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (BF16) {
        x[j * 8 + 2 * q] = __uint_as_float(w[q] << 16);
        x[j * 8 + 2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
      } else {
        x[j * 4 + q] = __uint_as_float(w[q]);
      }
    }
  }
}

// direct (non-TMA) load of this thread's vectors of a chunk, scalar loads, -inf past the row end;
// used only when rows are not 16-byte aligned (bulk copies need 16 B alignment and sizes)
template <bool BF16>
__device__ __forceinline__ void load_direct(const char* row, int chunk_base, int V, int tid,
                                            uint4 (&raw)[kVecPerThread]) {
  constexpr int EPV = Traits<BF16>::EPV;
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    const int e0 = chunk_base + (j * kConsumers + tid) * EPV;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = BF16 ? 0xff80ff80u : 0xff800000u;  // -inf
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      if (e0 + e < V) {
        if (BF16) {
          const uint32_t h = *reinterpret_cast<const unsigned short*>(row + (size_t)(e0 + e) * 2);
          const int q = e >> 1;
          w[q] = (e & 1) ? ((w[q] & 0x0000ffffu) | (h << 16)) : ((w[q] & 0xffff0000u) | h);
        } else {
          w[e] = *reinterpret_cast<const uint32_t*>(row + (size_t)(e0 + e) * 4);
        }
      }
    }
    raw[j] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// per-warp top-k state in shared memory (64-bit keys)
struct WarpTopk {
  unsigned long long buf[kSegBuf];  // candidates of the current row slice (appended; compacted)
  unsigned long long list[kMaxK];   // compacted top-k, sorted best first
  int cnt;                          // append cursor of the owner-lane expansion
  int pad[3];
};

// consumer-side shared state of a streaming CTA
struct __align__(16) ConsShared {
  unsigned long long tau;                                       // slice-wide bound hint (max over warps)
  __align__(16) unsigned pub[2][kConsumerWarps * kMaxK];        // slice start: top-j lane maxima per warp
  __align__(16) unsigned long long cl[kConsumerWarps * kMaxK];  // slice end: each warp's top-k
  __align__(16) float wmax[kConsumerWarps];                     // each warp's running max over the slice
  WarpTopk w[kConsumerWarps];
};

// Warp-level compaction: list <- top-k of buf[0..n) by rank counting (keys distinct); ranks >= n
// are sentinels.  The buffer then restarts from the list (caller sets its count to min(n, k)).
__device__ __forceinline__ void warp_compact(WarpTopk& w, int n, int k, int lane) {
  if (lane < k) w.list[lane] = kKeySentinel;
  __syncwarp();
  for (int e = lane; e < n; e += 32) {
    const unsigned long long key = w.buf[e];
    int rank = 0;
#pragma unroll 8
    for (int f = 0; f < n; ++f) rank += (w.buf[f] > key);
    if (rank < k) w.list[rank] = key;
  }
  __syncwarp();
  if (lane < k) w.buf[lane] = w.list[lane];
  __syncwarp();
}

// One 16 KiB chunk c of the slice [mlo, ...) of a row, by one consumer warp: the thread's vectors
// are `raw`; writes the (chunk, warp) softmax partial to msl[(c - mlo) * 8 + warp] and appends the
// chunk's top-k candidates to the warp buffer.  `stage` is the ring stage holding the chunk (TMA)
// or null (direct loads: `rowp` is the row).  `i` is the CTA's running chunk counter (parity of
// the slice-start publication buffer).
template <bool BF16, bool TMA>
__device__ __forceinline__ void consume_chunk(const Params& P, ConsShared& sh, float2* msl, const uint4 (&raw)[kVecPerThread],
                                              const char* stage, const char* rowp, int c, int mlo, int mhi, int i,
                                              int& wcnt, unsigned long long& bound, float& wrun) {
  constexpr int EPT = Traits<BF16>::EPT;
  constexpr int EPV = Traits<BF16>::EPV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = P.k, V = P.V, cpr = P.cpr;
  WarpTopk& W = sh.w[warp];
#ifndef CONSUME_EXPERIMENT
#define CONSUME_EXPERIMENT 0  // tools/ubench/consume.cu only: 1 stream only, 2 softmax only, 3 top-k only
#endif
  if (CONSUME_EXPERIMENT == 1) {
    if (lane == 0) msl[(c - mlo) * kConsumerWarps + warp] = make_float2(__uint_as_float(raw[0].x), 0.f);
    return;
  }
  CSTAMP(0 + 8 * (c - mlo));
  float x[EPT];
  unpack<BF16>(raw, x);
  const int cbase = c * P.chunk_elems;
  if (c == cpr - 1) {  // ragged last chunk: elements past the row end -> -inf
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (elem_index<BF16>(cbase, tid, e) >= V) x[e] = -INFINITY;
  }
  // ---- softmax partial of this (chunk, warp): max tree, 2 independent pair-sum chains ----
  float vm[kVecPerThread];
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    float a0 = fmaxf(x[j * EPV], x[j * EPV + 1]);
    float a1 = fmaxf(x[j * EPV + 2], x[j * EPV + 3]);
    if (EPV == 8) {
      a0 = fmaxf(a0, fmaxf(x[j * EPV + 4 % EPV], x[j * EPV + 5 % EPV]));
      a1 = fmaxf(a1, fmaxf(x[j * EPV + 6 % EPV], x[j * EPV + 7 % EPV]));
    }
    vm[j] = fmaxf(a0, a1);
  }
  const float m = fmaxf(fmaxf(vm[0], vm[1]), fmaxf(vm[2], vm[3]));
  const float Mw = warp_max_fast(m);
  CSTAMP(1 + 8 * (c - mlo));
  // exp2(x*log2e - M*log2e) on element pairs: FFMA2 + 2 MUFU + FADD2 (two pair accumulators)
  unsigned long long acc2[2] = {0ull, 0ull};
  if (Mw != -INFINITY && CONSUME_EXPERIMENT != 3) {
    const float ML = Mw * kLog2e;
    const unsigned long long l2e2 = f2pk(kLog2e, kLog2e), nml2 = f2pk(-ML, -ML);
#pragma unroll
    for (int e = 0; e < EPT; e += 2) {
      const unsigned long long y = ffma2(f2pk(x[e], x[e + 1]), l2e2, nml2);
      acc2[(e >> 1) & 1] = fadd2(acc2[(e >> 1) & 1], f2pk(ex2(f2lo(y)), ex2(f2hi(y))));
    }
  }
  const float sacc = warp_sum((f2lo(acc2[0]) + f2hi(acc2[0])) + (f2lo(acc2[1]) + f2hi(acc2[1])));
  if (lane == 0) msl[(c - mlo) * kConsumerWarps + warp] = make_float2(Mw, sacc);
  CSTAMP(2 + 8 * (c - mlo));
  if (CONSUME_EXPERIMENT == 2) return;

  // ---- top-k candidates of this warp-chunk ----
  // CTA-wide bound at the slice's first chunk: every warp publishes its top-j lane maxima
  // (j = max(ceil(k/8), 2) rounds of a warp max; ties keep their multiplicity); these 8j values are
  // distinct elements of the row, so their k-th largest v_k bounds the row's k-th best value from
  // below and key(v_k, INT_MAX) bounds the slice's k-th best key.  Later chunks run barrier-free
  // on the warp's own bound (tightened by compaction) and the CTA hint sh.tau.
  if (c == mlo) {
    const int jr = max((k + kConsumerWarps - 1) / kConsumerWarps, 2);
    unsigned* pub = sh.pub[i & 1];
    wrun = Mw;
    if (lane == 0) sh.wmax[warp] = -INFINITY;  // this slice's values are posted after the barrier below
    unsigned rem = (m == m) ? float_orderable(m) : 0u;
    for (int r = 0; r < jr; ++r) {
      const unsigned cur = __reduce_max_sync(kFull, rem);
      const unsigned bal = __ballot_sync(kFull, rem == cur);
      if (lane == __ffs(bal) - 1) rem = 0u;
      if (lane == 0) pub[warp * jr + r] = cur;
    }
    CSTAMP(3 + 8 * (c - mlo));
    consumer_sync();
    CSTAMP(4 + 8 * (c - mlo));
    const int np = kConsumerWarps * jr;  // multiple of 8
    unsigned vc = 0xffffffffu;
    if (np == 16) {  // k <= 16: all 16 values in registers (four broadcast 16-byte loads issued together)
      uint4 v4[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) v4[o] = *reinterpret_cast<const uint4*>(pub + 4 * o);
      const unsigned u = lane < 16 ? pub[lane] : 0u;
      int gt = 0;
#pragma unroll
      for (int o = 0; o < 4; ++o) gt += (v4[o].x > u) + (v4[o].y > u) + (v4[o].z > u) + (v4[o].w > u);
      if (lane < 16 && gt < k) vc = u;
    } else {
      for (int e = lane; e < np; e += 32) {
        const unsigned u = pub[e];
        int gt = 0;
        for (int o = 0; o < np; o += 4) {
          const uint4 v4 = *reinterpret_cast<const uint4*>(pub + o);  // broadcast reads
          gt += (v4.x > u) + (v4.y > u) + (v4.z > u) + (v4.w > u);
        }
        if (gt < k && u < vc) vc = u;
      }
    }
    const unsigned vk = __reduce_min_sync(kFull, vc);
    if (vk != 0u && vk != 0xffffffffu) {  // 0: NaN maxima among the top k (row flagged; no bound)
      const unsigned long long b0 = ((unsigned long long)vk << 32) | 0x80000000ull;  // (v_k, INT_MAX)
      if (b0 > bound) bound = b0;
    }
    if (lane == 0) *reinterpret_cast<volatile float*>(&sh.wmax[warp]) = wrun;
  } else if (k <= kConsumerWarps) {
    // later chunks: every warp's running max over the slice is an element of the row (distinct
    // elements for distinct warps), so the k-th largest of the 8 posted maxima bounds the slice's
    // k-th best value from below; stale or unposted entries are smaller (still valid) or -inf
    wrun = fmaxf(wrun, Mw);
    if (lane == 0) *reinterpret_cast<volatile float*>(&sh.wmax[warp]) = wrun;
    float wv[kConsumerWarps];
    asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(wv[0]), "=f"(wv[1]), "=f"(wv[2]), "=f"(wv[3]) : "r"(smem_u32(&sh.wmax[0])));
    asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(wv[4]), "=f"(wv[5]), "=f"(wv[6]), "=f"(wv[7]) : "r"(smem_u32(&sh.wmax[4])));
    float vkth;
    if (k == kConsumerWarps) {
      vkth = fminf(fminf(fminf(wv[0], wv[1]), fminf(wv[2], wv[3])), fminf(fminf(wv[4], wv[5]), fminf(wv[6], wv[7])));
    } else {
      vkth = INFINITY;  // the smallest value with fewer than k larger entries
#pragma unroll
      for (int x = 0; x < kConsumerWarps; ++x) {
        int gt = 0;
#pragma unroll
        for (int y = 0; y < kConsumerWarps; ++y) gt += (wv[y] > wv[x]) || (wv[y] == wv[x] && y < x);
        if (gt < k) vkth = fminf(vkth, wv[x]);
      }
    }
    if (vkth > -INFINITY && vkth == vkth) {
      const unsigned long long b0 = ((unsigned long long)float_orderable(vkth) << 32) | 0x80000000ull;
      if (b0 > bound) bound = b0;
    }
  }
  {
    // barrier-free CTA bound: every warp posts its k-th best after each compaction (a lower
    // bound of the slice's k-th best) with a shared atomic max; all warps adopt the maximum
    const unsigned long long tt = *reinterpret_cast<volatile unsigned long long*>(&sh.tau);
    if (tt > bound) bound = tt;
  }
  if (CONSUME_EXPERIMENT == 4) {  // ubench only: an oracle-quality bound from the first chunk on
    const unsigned long long b9 = ((unsigned long long)float_orderable(9.0f) << 32) | 0x80000000ull;
    if (b9 > bound) bound = b9;
  }
  float bv = bound ? tk_val(bound) : -INFINITY;
  CSTAMP(5 + 8 * (c - mlo));
  CCOUNT(0, 1);
  bool done = false;
  if (TMA && __any_sync(kFull, m >= bv)) {
    // owner-lane expansion: a lane re-reads its qualifying vectors from the still-held stage and
    // marks the elements reaching the bound; the candidates are appended at positions from a
    // warp-local shared cursor (the buffer is compacted by rank later, so order is irrelevant)
    CCOUNT(1, 1);
    uint32_t cm = 0u;
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      if (vm[j] >= bv) {
        const uint4 q = reinterpret_cast<const uint4*>(stage)[j * kConsumers + tid];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          const float xv = BF16 ? __uint_as_float((e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16))
                                : __uint_as_float(w[e]);
          if (xv >= bv && elem_index<BF16>(cbase, tid, j * EPV + e) < V) cm |= 1u << (j * EPV + e);
        }
      }
    }
    const int n = __popc(cm);
    const int tot = __reduce_add_sync(kFull, (unsigned)n);
    if (wcnt + tot <= kSegBuf) {
      if (lane == 0) W.cnt = wcnt;
      __syncwarp();
      if (n) {
        int pos = atomicAdd(&W.cnt, n);
        while (cm) {
          const int b = __ffs(cm) - 1;
          cm &= cm - 1u;
          const int j = b / EPV, e = b % EPV;
          const uint4 q = reinterpret_cast<const uint4*>(stage)[j * kConsumers + tid];
          const uint32_t wv = (BF16 ? e >> 1 : e) == 0 ? q.x : (BF16 ? e >> 1 : e) == 1 ? q.y : (BF16 ? e >> 1 : e) == 2 ? q.z : q.w;
          const float xv = BF16 ? __uint_as_float((e & 1) ? (wv & 0xffff0000u) : (wv << 16)) : __uint_as_float(wv);
          W.buf[pos++] = tk_key(xv, elem_index<BF16>(cbase, tid, b));
        }
      }
      __syncwarp();
      wcnt += tot;
      CCOUNT(2, tot);
      done = true;
    }
  }
  if (!done && __any_sync(kFull, m >= bv)) {  // most chunks of a long slice have no candidate at all
    CCOUNT(1, 1);
    // vectors whose max reaches the bound are expanded cooperatively: each group of EPV lanes
    // takes one such vector (its elements re-read from the still-held ring stage), compares them
    // with the bound and appends the survivors at ballot-prefix positions
    constexpr int G = 32 / EPV;  // vectors per pass
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      unsigned bal = __ballot_sync(kFull, vm[j] >= bv);
      while (bal) {
        if (wcnt > kSegBuf - 32) {  // keep room for a full pass: compact, tighten, re-filter
          CCOUNT(3, 1);
          __syncwarp();
          warp_compact(W, wcnt, k, lane);
          wcnt = k;
          if (W.list[k - 1] > bound) bound = W.list[k - 1];
          if (lane == 0) atomicMax(&sh.tau, W.list[k - 1]);
          bv = tk_val(bound);
          bal &= __ballot_sync(kFull, vm[j] >= bv);
          if (!bal) break;
        }
        unsigned bb = bal;
        for (int g = 0; g < lane / EPV; ++g) bb &= bb - 1u;
        const int L = bb ? __ffs(bb) - 1 : -1;  // owner lane of this group's vector
#pragma unroll
        for (int g = 0; g < G; ++g) bal &= bal - 1u;
        bool q = false;
        float v = -INFINITY;
        int idx = 0;
        if (L >= 0) {
          const int tl = warp * 32 + L;  // the owner's consumer thread id
          const int e = j * EPV + lane % EPV;
          idx = elem_index<BF16>(cbase, tl, e);
          if (idx < V) {  // past the row end: stale stage bytes, never a candidate
            const char* sp = TMA ? stage + ((size_t)(j * kConsumers + tl) * EPV + (e % EPV)) * (BF16 ? 2 : 4)
                                 : rowp + (size_t)idx * (BF16 ? 2 : 4);
            v = BF16 ? __uint_as_float((uint32_t)(*reinterpret_cast<const unsigned short*>(sp)) << 16)
                     : *reinterpret_cast<const float*>(sp);
          }
          q = v >= bv;  // NaN never qualifies (the row merge flags it)
        }
        const unsigned qb = __ballot_sync(kFull, q);
        if (q) W.buf[wcnt + __popc(qb & ((1u << lane) - 1u))] = tk_key(v, idx);
        wcnt += __popc(qb);
        CCOUNT(2, __popc(qb));
        CCOUNT(5, 1);
      }
    }
  }
  CSTAMP(6 + 8 * (c - mlo));
  if (wcnt >= 2 * k && c + 1 < mhi) {  // keep the warp's buffer short
    CCOUNT(4, 1);
    __syncwarp();
    warp_compact(W, wcnt, k, lane);
    wcnt = k;
    if (W.list[k - 1] > bound) bound = W.list[k - 1];
    if (lane == 0) atomicMax(&sh.tau, W.list[k - 1]);
  }
  CSTAMP(7 + 8 * (c - mlo));
}

// Slice end, part 1 (every consumer warp): the warp's padded top-k into sh.cl, then a consumer
// barrier.  Padding keys are distinct and below every real key (value -inf, index > INT_MAX).
__device__ __forceinline__ void slice_end_post(ConsShared& sh, int k, int& wcnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpTopk& W = sh.w[warp];
  if (wcnt > k) {
    warp_compact(W, wcnt, k, lane);
    wcnt = k;
  }
  CSTAMP(40);
  if (lane < k) sh.cl[warp * k + lane] = lane < wcnt ? W.buf[lane] : kKeySentinel - 1 - (warp * k + lane);
  wcnt = 0;
  consumer_sync();
  CSTAMP(41);
}

// Slice end, part 2 (after slice_end_post): the CTA's top-k of the slice by a rank merge of the
// nl = 8k entries (broadcast 16-byte reads), emitted as out_key(rank, key) for rank < k, plus an
// even-k padding key at rank k; and per chunk of the slice the 8 warps' (M_w, s_w) combined in
// warp order (fixed association: a function of the chunk alone), emitted as out_ms(cc, M_c, S_c).
template <class KeyOut, class MsOut>
__device__ __forceinline__ void slice_end_merge(const ConsShared& sh, const float2* msl, int k, int nch, KeyOut out_key,
                                                MsOut out_ms) {
  const int tid = threadIdx.x;
  const int nl = kConsumerWarps * k;  // even
  if (tid < nl) {
    const unsigned long long key = sh.cl[tid];
    const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(sh.cl);
    int r0 = 0, r1 = 0;
    if (k <= kConsumerWarps) {
      // k <= 8: at most 64 entries, all 32 broadcast loads issued back to back (no loop-carried
      // latency), the padding beyond nl never counted
#pragma unroll
      for (int f = 0; f < kConsumerWarps * kConsumerWarps / 2; ++f) {
        const ulonglong2 v = c2[f];
        r0 += (2 * f < nl && v.x > key);
        r1 += (2 * f + 1 < nl && v.y > key);
      }
    } else {
#pragma unroll 4
      for (int f = 0; f < nl / 2; ++f) {
        const ulonglong2 v = c2[f];
        r0 += (v.x > key);
        r1 += (v.y > key);
      }
    }
    const int rank = r0 + r1;
    if (rank < k) out_key(rank, key);
  }
  if ((k & 1) && tid == 0) out_key(k, kKeySentinel - 1000);  // even-k padding slot
  for (int cc = kConsumers - 1 - tid; cc < nch; cc += kConsumers) {
    const float2* pw = msl + cc * kConsumerWarps;
    float Mc = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) Mc = fmaxf(Mc, pw[w].x);
    const float MLc = Mc * kLog2e;
    float Sc = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      const float2 v = pw[w];
      if (v.y != 0.f || isnan(v.y)) Sc += v.y * ex2(fmaf(v.x, kLog2e, -MLc));
    }
    out_ms(cc, Mc, Sc);
  }
}

// kp = k rounded up to even, so every list is a multiple of 16 bytes
__host__ __device__ inline int list_stride(int k) { return (k + 1) & ~1; }

// Row merge by one warp (A1 finish + A2): M, Z from the row's cpr per-chunk partials (fixed
// lane-strided association: a function of cpr only); T = the best k-th entry over the t slice
// lists (each list is its slice's top-k, so T bounds the row's k-th best key from below); the
// entries >= T ranked among themselves; the top k emitted as emit(rank, tok, p, cum) with
// p = exp(x - M)/Z (tau = 1) and cum = pc * p (Eq.(3)).  ms(c) and key(e) read the
// partials (any memory space); surv is a per-warp scratch of >= k + (t-1)(k-1) keys.  Returns
// false if the row holds NaN/+inf or no finite logit (Q23).
template <class MsAt, class KeyAt, class Emit>
__device__ __forceinline__ bool merge_row(int k, int cpr, int t, float pc, MsAt ms, KeyAt key_at,
                                          unsigned long long* surv, Emit emit) {
  const int lane = threadIdx.x & 31;
  const float4 v0 = lane < cpr ? ms(lane) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const float4 v1 = lane + 32 < cpr ? ms(lane + 32) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const float M = warp_max_fast(fmaxf(v0.x, v1.x));
  const float ML = M * kLog2e;
  float z = 0.f;
  z += (v0.y != 0.f || isnan(v0.y)) ? v0.y * ex2(fmaf(v0.x, kLog2e, -ML)) : 0.f;
  z += (v1.y != 0.f || isnan(v1.y)) ? v1.y * ex2(fmaf(v1.x, kLog2e, -ML)) : 0.f;
  const float Z = warp_sum(z);
  const float rZ = __frcp_rn(Z);  // correctly rounded 1/Z (no division slow path)
  const int kp = list_stride(k);
  const unsigned long long tail = lane < t ? key_at(lane * kp + k - 1) : 0ull;
  const unsigned th = __reduce_max_sync(kFull, (unsigned)(tail >> 32));
  const unsigned tl = __reduce_max_sync(kFull, (unsigned)(tail >> 32) == th ? (unsigned)tail : 0u);
  const unsigned long long T = ((unsigned long long)th << 32) | tl;
  const int nkey = t * kp;  // the padding slot of an odd k holds a key below every real one
  int ns = 0;
  for (int e0 = 0; e0 < nkey; e0 += 32) {
    const int e = e0 + lane;
    const unsigned long long key = e < nkey ? key_at(e) : 0ull;
    const bool sv = e < nkey && key >= T;
    const unsigned bal = __ballot_sync(kFull, sv);
    if (sv) surv[ns + __popc(bal & ((1u << lane) - 1u))] = key;
    ns += __popc(bal);
  }
  __syncwarp();
  auto out = [&](unsigned long long key, int rank) {
    const float v = tk_val(key);
    const float pj = ex2(fmaf(v, kLog2e, -ML)) * rZ;  // p = exp(x - M) / Z   (tau = 1, Q10)
    emit(rank, tk_idx(key), pj, pc * pj);             // Eq.(3)
  };
  if (ns <= 32) {
    // one survivor per lane; rank by broadcast compares
    const unsigned long long mine = lane < ns ? surv[lane] : 0ull;
    int rank = 0;
#pragma unroll 8
    for (int q = 0; q < ns; ++q) rank += (__shfl_sync(kFull, mine, q) > mine);
    if (lane < ns && rank < k) out(mine, rank);
  } else {
    for (int s0 = lane; s0 < ns; s0 += 32) {
      const unsigned long long key = surv[s0];
      int r0 = 0, r1 = 0;
      int q = 0;
      for (; q + 1 < ns; q += 2) {
        r0 += (surv[q] > key);
        r1 += (surv[q + 1] > key);
      }
      if (q < ns) r0 += (surv[q] > key);
      const int rank = r0 + r1;
      if (rank < k) out(key, rank);
    }
  }
  __syncwarp();
  return (Z >= 1.0f) && !isinf(Z) && !isnan(M);
}

// Row merge by a k-round tournament (A1 finish + A2), for t <= 32 slice lists each sorted best
// first and held in shared memory at keys + m * kp: lane m holds the head of list m and the next
// entry; every round the warp's maximum key (two REDUX: value word, then index word among the
// value's holders) is the row's next best, and its lane advances branch-free (every lane reloads
// its next entry from a precomputed 32-bit shared address).  Same outputs as merge_row.
template <class MsAt, class Emit>
__device__ __forceinline__ bool merge_row_tournament(int k, int cpr, int t, float pc, MsAt ms,
                                                     const unsigned long long* keys, Emit emit) {
  const int lane = threadIdx.x & 31;
  const int kp = list_stride(k);
  const float4 v0 = lane < cpr ? ms(lane) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const float4 v1 = lane + 32 < cpr ? ms(lane + 32) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const bool own = lane < t;
  const uint32_t base = smem_u32(keys + (own ? lane : 0) * kp);
  unsigned long long cur = own ? keys[lane * kp] : 0ull;
  unsigned long long nxt = own && k > 1 ? keys[lane * kp + 1] : 0ull;
  int h = 1;  // index of nxt in the lane's list
  const float M = warp_max_fast(fmaxf(v0.x, v1.x));
  const float ML = M * kLog2e;
  float z = 0.f;
  z += (v0.y != 0.f || isnan(v0.y)) ? v0.y * ex2(fmaf(v0.x, kLog2e, -ML)) : 0.f;
  z += (v1.y != 0.f || isnan(v1.y)) ? v1.y * ex2(fmaf(v1.x, kLog2e, -ML)) : 0.f;
  const float Z = warp_sum(z);
  const float rZ = __frcp_rn(Z);  // correctly rounded 1/Z (no division slow path)
  unsigned long long mine = 0ull;  // lane r keeps the r-th best key
  for (int r = 0; r < k; ++r) {
    // one warp max on the value word; the low (index) word only when values tie (rare)
    const unsigned hv = (unsigned)(cur >> 32);
    const unsigned hi = __reduce_max_sync(kFull, hv);
    unsigned bal = __ballot_sync(kFull, hv == hi);
    if (bal & (bal - 1u)) {
      const unsigned lo = __reduce_max_sync(kFull, hv == hi ? (unsigned)cur : 0u);
      bal = __ballot_sync(kFull, hv == hi && (unsigned)cur == lo);
    }
    const int wl = __ffs(bal) - 1;  // keys are distinct: exactly one winner
    const unsigned long long win = ((unsigned long long)hi << 32) | (unsigned)__shfl_sync(kFull, (unsigned)cur, wl);
    mine = lane == r ? win : mine;
    const bool adv = lane == wl;
    cur = adv ? nxt : cur;
    h += adv ? 1 : 0;
    unsigned long long ld;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ld) : "r"(base + 8u * (uint32_t)min(h, k - 1)));
    nxt = adv ? (h < k ? ld : 0ull) : nxt;
  }
  if (lane < k) {
    const float v = tk_val(mine);
    const float pj = ex2(fmaf(v, kLog2e, -ML)) * rZ;  // p = exp(x - M) / Z   (tau = 1, Q10)
    emit(lane, tk_idx(mine), pj, pc * pj);            // Eq.(3)
  }
  __syncwarp();
  return (Z >= 1.0f) && !isinf(Z) && !isnan(M);
}

// Row merge by threshold + rank (A1 finish + A2) for t <= 32 slice lists, each the top-k of its
// slice sorted best first, in shared memory at keys + m * kp (kp = list_stride(k)).  No sequential
// rounds: T = max(best k-th entry over the lists, k-th best list head) is a lower bound of the
// row's k-th best key (each bounds it: a list's k-th entry is the k-th best of a subset; the k
// largest heads are k distinct elements); the survivors (entries >= T, typically ~k) are compacted
// and ranked by counting with broadcast loads.  Z from the cpr per-chunk partials as merge_row.
// `surv` is a per-warp scratch of >= t * k keys.  Same outputs as merge_row.
template <class MsAt, class Emit>
__device__ __forceinline__ bool merge_row_rank(int k, int cpr, int t, float pc, MsAt ms,
                                               const unsigned long long* keys, unsigned long long* surv, Emit emit) {
  const int lane = threadIdx.x & 31;
  const int kp = list_stride(k);
  const bool own = lane < t;
  const unsigned long long* my = keys + lane * kp;
  const unsigned long long head = own ? my[0] : 0ull, tail = own ? my[k - 1] : 0ull;
  const float4 v0 = lane < cpr ? ms(lane) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const float4 v1 = lane + 32 < cpr ? ms(lane + 32) : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  // (1) thresholds: the best tail (two reductions) and the k-th best head (rank among the heads)
  const unsigned th = __reduce_max_sync(kFull, (unsigned)(tail >> 32));
  const unsigned tl = __reduce_max_sync(kFull, (unsigned)(tail >> 32) == th ? (unsigned)tail : 0u);
  unsigned long long T = ((unsigned long long)th << 32) | tl;
  if (t >= k) {
    int hr = 0;  // heads better than mine
    for (int m = 0; m < t; ++m) hr += keys[m * kp] > head;
    const unsigned bal = __ballot_sync(kFull, own && hr == k - 1);
    const unsigned long long Th = __shfl_sync(kFull, head, __ffs(bal) - 1);
    if (Th > T) T = Th;
  }
  // (2) softmax normaliser (independent of the top-k work)
  const float M = warp_max_fast(fmaxf(v0.x, v1.x));
  const float ML = M * kLog2e;
  float z = 0.f;
  z += (v0.y != 0.f || isnan(v0.y)) ? v0.y * ex2(fmaf(v0.x, kLog2e, -ML)) : 0.f;
  z += (v1.y != 0.f || isnan(v1.y)) ? v1.y * ex2(fmaf(v1.x, kLog2e, -ML)) : 0.f;
  const float Z = warp_sum(z);
  const float rZ = __frcp_rn(Z);  // correctly rounded 1/Z (no division slow path)
  // (3) survivors, compacted by ballots over the entry index j (lists are sorted: entries < T end
  // a list's survivors, so the loop stops at the first j without any)
  int ns = 0;
  for (int j = 0; j < k; ++j) {
    const unsigned long long key = own ? my[j] : 0ull;
    const bool sv = own && key >= T;
    const unsigned bal = __ballot_sync(kFull, sv);
    if (!bal) break;
    if (sv) surv[ns + __popc(bal & ((1u << lane) - 1u))] = key;
    ns += __popc(bal);
  }
  __syncwarp();
  // (4) exact ranks among the survivors (keys distinct); the top k emitted
  auto out = [&](unsigned long long key, int rank) {
    const float v = tk_val(key);
    const float pj = ex2(fmaf(v, kLog2e, -ML)) * rZ;  // p = exp(x - M) / Z   (tau = 1, Q10)
    emit(rank, tk_idx(key), pj, pc * pj);             // Eq.(3)
  };
  for (int s0 = lane; s0 < ns; s0 += 32) {
    const unsigned long long key = surv[s0];
    int r0 = 0, r1 = 0, q = 0;
    for (; q + 1 < ns; q += 2) {
      r0 += surv[q] > key;
      r1 += surv[q + 1] > key;
    }
    if (q < ns) r0 += surv[q] > key;
    if (r0 + r1 < k) out(key, r0 + r1);
  }
  __syncwarp();
  return (Z >= 1.0f) && !isinf(Z) && !isnan(M);
}

}  // namespace smart
