// expand.cu — the per-layer kernel: K1 `smart_expand_step` (A1 top-k + softmax of every frontier
// row; A2 path score cum = cum(parent) * p, Eq.(3)) with the
// layer's selection A3-A6 fused into the tail of the last CTA (single rank).
//
// Design:
//  * HBM stream, TMA-staged: the frontier rows are cut into 16 KiB chunks; a persistent grid
//    (#SMs x 2 CTAs) takes balanced contiguous ranges of (row, chunk) units.  A producer warp
//    bulk-copies chunks (cp.async.bulk + mbarrier tx count) into a 6-stage shared-memory ring;
//    8 consumer warps read 16-byte vectors from it.
//  * softmax: each consumer warp reduces its 1024 (bf16) / 512 (fp32) elements of a chunk to
//    (max, sum exp) with a fixed shuffle tree; the row merge combines the cpr x 8 partials in
//    fixed order, so Z is bit-identical for any grid size or sharding.
//  * top-k (exact, ties -> lower index): keys are 64-bit (orderable value | ~index), so one
//    compare orders two candidates.  Per warp and segment (consecutive chunks of one row in one
//    CTA) a running lower bound of the k-th best key is kept: at the segment's first chunk it is
//    the k-th largest lane-maximum value (k rounds of a one-instruction warp max), later tightened
//    by compactions and a CTA-wide hint.  Only the 16-byte vectors whose max reaches the bound
//    are scanned; qualifying elements are appended to a per-warp buffer in shared memory, which
//    is compacted to its top-k (rank counting) when full and at the segment end.
//  * the CTA that completes a row's last chunk merges that row (Z, exact top-k, p, cum); the CTA
//    that merges the layer's last row runs the selection for the whole batch (select_core.cuh).
//    Arrival counters use one acq_rel atomic per CTA after a CTA barrier (no per-thread fences).
#include "select_core.cuh"
#include "stream.cuh"

namespace smart {

namespace {

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

// logits row of frontier row `row` (layer parity `par`); rows [row0, row0 + kStageRows) use the
// frontier entries staged in shared memory
__device__ __forceinline__ const char* row_ptr(const Params& P, int par, const char* base, long long ld_bytes,
                                              int row, const int2* rfe, int row0) {
  if (P.row_mode == SMART_ROWS_NODE) {
    const int2 fe = (row - row0 < kStageRows) ? rfe[row - row0] : P.fr[par][row];
    return base + ((long long)fe.x * P.T + fe.y) * ld_bytes;
  }
  return base + (long long)row * ld_bytes;
}

// per-warp top-k state in shared memory (64-bit keys)
struct WarpTopk {
  unsigned long long buf[kSegBuf];  // candidates of the current segment (appended; compacted)
  unsigned long long list[kMaxK];   // compacted top-k, sorted best first
};

struct ExpandShared {
  int2 rfe[kStageRows];  // frontier entries of the CTA's first rows
  unsigned pub[2][kConsumerWarps * 4];  // per chunk (double-buffered): top-j lane maxima of each warp
  unsigned long long cl[kConsumerWarps * kMaxK];  // segment end: each warp's top-k (distinct sentinels)
  int last_layer;
  WarpTopk w[kConsumerWarps];
};

// row-merge staging, carved from the dynamic shared memory after ExpandShared (sized by cpr, k)
struct MergeStage {
  unsigned long long* keys;  // [cpr * k] segment lists (valid at segment-start chunks)
  unsigned long long* surv;  // [cpr * k] survivors of the threshold
};

__host__ __device__ inline size_t merge_stage_bytes(int cpr, int k) { return (size_t)cpr * k * 16; }

__device__ inline MergeStage merge_stage(char* base, int cpr, int k) {
  MergeStage m;
  m.keys = reinterpret_cast<unsigned long long*>(base);
  m.surv = m.keys + (size_t)cpr * k;
  return m;
}

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

// ---- row merge by one warp of the CTA that completed the row (no CTA barriers) ----
// One load wave (partials, segment lengths, segment lists, frontier entry and its cum), then:
// M = max, Z = sum s*exp(m - M) with an association fixed by cpr; T = the best k-th entry over
// the segment lists (a lower bound of the row's k-th best key, every list holding its segment's
// top-k); the entries >= T are ranked among themselves and the top k written with p and cum.
__device__ void merge_row_warp(const Params& P, int layer, int par, int row, MergeStage st) {
  const int lane = threadIdx.x & 31;
  const bool sp = (row == 0 && lane == 0);
  stamp(P, sp, 24);
  const int k = P.k, cpr = P.cpr;
  const int npart = cpr * kConsumerWarps;  // <= 512
  const int nkey = cpr * k;                // <= 2048
  // ---- load wave ----
  const float2* ms = P.ms + (size_t)row * npart;
  float2 part[kMaxCpr * kConsumerWarps / 32];
#pragma unroll
  for (int t = 0; t < kMaxCpr * kConsumerWarps / 32; ++t)
    part[t] = (lane + 32 * t < npart) ? __ldcg(&ms[lane + 32 * t]) : make_float2(-INFINITY, 0.f);
  int* sl = P.seglen + (size_t)row * cpr;
  const int sl0 = lane < cpr ? __ldcg(&sl[lane]) : 0;
  const int sl1 = lane + 32 < cpr ? __ldcg(&sl[lane + 32]) : 0;
  const unsigned long long* sk = P.segkey + (size_t)row * nkey;
  for (int e0 = 0; e0 < nkey; e0 += 256) {  // batches of independent loads, then the stores
    unsigned long long v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 32 + lane;
      v[u] = e < nkey ? __ldcg(&sk[e]) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 32 + lane;
      if (e < nkey) st.keys[e] = v[u];
    }
  }
  int2 fe = make_int2(0, 0);
  float pc = 0.f;
  if (lane == 0) {
    fe = P.fr[par][row];
    pc = P.fr_cum[par][row];
  }
  if (lane < cpr) sl[lane] = 0;  // self-cleaning for the next use
  if (lane + 32 < cpr) sl[lane + 32] = 0;
  stamp(P, sp, 25);
  // ---- (1) softmax normaliser ----
  float m = -INFINITY;
#pragma unroll
  for (int t = 0; t < kMaxCpr * kConsumerWarps / 32; ++t) m = fmaxf(m, part[t].x);
  const float M = warp_max_fast(m);
  const float ML = M * kLog2e;
  float z = 0.f;
#pragma unroll
  for (int t = 0; t < kMaxCpr * kConsumerWarps / 32; ++t) {
    const float2 v = part[t];
    if (v.y != 0.f || isnan(v.y)) z += v.y * ex2(fmaf(v.x, kLog2e, -ML));
  }
  const float Z = warp_sum(z);
  stamp(P, sp, 26);
  // ---- (2) threshold T = max over segments of their k-th entry ----
  const unsigned long long v0 = __ballot_sync(kFull, sl0 > 0), v1 = __ballot_sync(kFull, sl1 > 0);
  __syncwarp();  // st.keys visible
  unsigned long long tail = 0ull;
  if (sl0 > 0) tail = st.keys[lane * k + k - 1];
  if (sl1 > 0 && st.keys[(lane + 32) * k + k - 1] > tail) tail = st.keys[(lane + 32) * k + k - 1];
  const unsigned th = __reduce_max_sync(kFull, (unsigned)(tail >> 32));
  const unsigned tl = __reduce_max_sync(kFull, (unsigned)(tail >> 32) == th ? (unsigned)tail : 0u);
  const unsigned long long T = ((unsigned long long)th << 32) | tl;
  stamp(P, sp, 27);
  // ---- (3) survivors (entries >= T of existing segments), compacted by ballot ----
  const unsigned kmag = 0xffffffffu / (unsigned)k + 1u;  // e / k == umulhi(e, kmag) (k >= 2, e < 2^16)
  int ns = 0;
  for (int e0 = 0; e0 < nkey; e0 += 32) {
    const int e = e0 + lane;
    bool sv = false;
    unsigned long long key = 0ull;
    if (e < nkey) {
      const int c = (k == 1) ? e : (int)__umulhi((unsigned)e, kmag);
      const bool valid = c < 32 ? ((v0 >> c) & 1ull) : ((v1 >> (c - 32)) & 1ull);
      if (valid) {
        key = st.keys[e];
        sv = key >= T;
      }
    }
    const unsigned bal = __ballot_sync(kFull, sv);
    if (sv) st.surv[ns + __popc(bal & ((1u << lane) - 1u))] = key;
    ns += __popc(bal);
  }
  __syncwarp();
  stamp(P, sp, 28);
  // ---- (4) exact top-k among the survivors by rank; A1 p and A2 cum ----
  fe.x = __shfl_sync(kFull, fe.x, 0);
  fe.y = __shfl_sync(kFull, fe.y, 0);
  pc = __shfl_sync(kFull, pc, 0);
  for (int s0 = lane; s0 < ns; s0 += 32) {
    const unsigned long long key = st.surv[s0];
    int r0 = 0, r1 = 0;
    int t = 0;
    for (; t + 1 < ns; t += 2) {
      r0 += (st.surv[t] > key);
      r1 += (st.surv[t + 1] > key);
    }
    if (t < ns) r0 += (st.surv[t] > key);
    const int rank = r0 + r1;
    if (rank < k) {
      const float v = tk_val(key);
      const float pj = ex2(fmaf(v, kLog2e, -ML)) / Z;  // p = exp(x - M) / Z   (tau = 1, Q10)
      Cand cd;
      cd.tok = tk_idx(key);
      cd.p = pj;
      cd.cum = pc * pj;  // Eq.(3)
      cd.parent = fe.y;
      P.cand[((size_t)(layer - 1) * P.cap_rows + row) * k + rank] = cd;
    }
  }
  stamp(P, sp, 29);
  if (lane == 0) {
    P.cand_rs[(size_t)(layer - 1) * P.cap_rows + row] = make_int2(fe.x, row - P.fr_off[par][fe.x]);
    P.rowstat[row] = make_float2(M, Z);
    if (!(Z >= 1.0f) || isinf(Z) || isnan(M)) atomicOr(P.err, kErrDraftNaN);  // Q23
    P.row_done[row] = 0;
  }
  __syncwarp();
  stamp(P, sp, 30);
}

template <bool BF16, bool TMA>
__global__ void __launch_bounds__(kLayerThreads, 2)
layer_kernel(Params P, int layer, const char* __restrict__ logits, long long ld_bytes, int fuse_select) {
  constexpr int EPT = Traits<BF16>::EPT;
  constexpr int EPV = Traits<BF16>::EPV;
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;
  StreamPipe& pipe = *reinterpret_cast<StreamPipe*>(dsm + kStages * kChunkBytes);
  ExpandShared& sh = *reinterpret_cast<ExpandShared*>(dsm + kStages * kChunkBytes + sizeof(StreamPipe));
  const MergeStage mst =
      merge_stage(dsm + kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(ExpandShared), P.cpr, P.k);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    mbar_fence_init();
    sh.last_layer = 0;
  }
  tl_start(P, 32 + layer);
  pdl_wait();
  pdl_trigger();
  tl_start(P, layer);
  if (tid == 0) {
    probe_min(P, 0);
    probe_max(P, 1);
  }
  const int R = *P.fr_total[par];
  const bool t0 = (blockIdx.x == 0 && tid == 0);
  gstamp(P, t0, 16);
  if (R == 0) {
    // A_{l-1} is empty for every request: the step has terminated at this layer
    if (fuse_select && blockIdx.x == 0 && tid == 0) *P.fr_total[layer & 1] = 0;
    return;
  }
  const int k = P.k, cpr = P.cpr, CE = P.chunk_elems, V = P.V;
  const long long row_bytes = (long long)V * (BF16 ? 2 : 4);
  const RowRange rr = cta_range_min(R * cpr, P.min_units);
  if (rr.lo >= rr.hi) return;
  // the CTA's frontier entries, staged once (no dependent global load per chunk)
  const int row0 = rr.lo / cpr;
  const int nstage = min((rr.hi - 1) / cpr - row0 + 1, kStageRows);
  if (tid < nstage) sh.rfe[tid] = P.fr[par][row0 + tid];
  __syncthreads();
  gstamp(P, t0, 17);

  if (warp == kConsumerWarps) {  // ---- producer warp ----
    gstamp(P, blockIdx.x == 0 && lane == 0, 27);
    if (TMA && lane == 0)
      produce(pipe, ring, rr, cpr, row_bytes, [&](int row) { return row_ptr(P, par, logits, ld_bytes, row, sh.rfe, row0); });
    return;
  }

  // ---- consumer warps ----
  WarpTopk& W = sh.w[warp];
  int wcnt = 0;  // entries in W.buf (warp-uniform)
  int i = 0;
  int q = rr.lo;
  int row = row0, c0 = rr.lo - row0 * cpr;
  while (q < rr.hi) {
    const int nch = min(cpr - c0, rr.hi - q);
    unsigned long long bound = 0ull;  // lower bound of the segment's k-th best key
    for (int c = c0; c < c0 + nch; ++c, ++i) {
      uint4 raw[kVecPerThread];
      const int s = (int)(i % kStages);
      if (TMA) {
        mbar_wait(&pipe.full[s], (uint32_t)((i / kStages) & 1));
        gstamp(P, t0 && i < 2, 18 + 3 * (int)i);
        stamp(P, t0 && i == 0, 0);
        const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * kChunkBytes);
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) raw[j] = st[j * kConsumers + tid];
      } else {
        load_direct<BF16>(row_ptr(P, par, logits, ld_bytes, row, sh.rfe, row0), c * CE, V, tid, raw);
      }
      float x[EPT];
      unpack<BF16>(raw, x);
      stamp(P, t0 && i == 0, 1);
      const int cbase = c * CE;
      if (c == cpr - 1) {  // ragged last chunk: elements past the row end -> -inf
#pragma unroll
        for (int n = 0; n < EPT; ++n)
          if (elem_index<BF16>(cbase, tid, n) >= V) x[n] = -INFINITY;
      }
      // ---- softmax partial of this (chunk, warp): max tree, 4 independent sum chains ----
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
      stamp(P, t0 && i == 0, 2);
      const float Mw = warp_max_fast(m);
      stamp(P, t0 && i == 0, 3);
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      if (Mw != -INFINITY) {
        const float ML = Mw * kLog2e;
#pragma unroll
        for (int n = 0; n < EPT; ++n) s4[n & 3] += ex2(fmaf(x[n], kLog2e, -ML));
      }
      const float sacc = warp_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
      if (lane == 0) P.ms[((size_t)row * cpr + c) * kConsumerWarps + warp] = make_float2(Mw, sacc);
      stamp(P, t0 && i == 0, 4);
      gstamp(P, t0 && i < 2, 19 + 3 * (int)i);

      // ---- top-k candidates of this warp-chunk ----
      // CTA-wide bound for this chunk: every warp publishes its top-j lane maxima (j = ceil(k/8),
      // one lane per round, so ties keep their multiplicity); these 8j values are distinct
      // elements of the row, so their k-th largest v_k bounds the row's k-th best value from
      // below and key(v_k, INT_MAX) bounds the segment's k-th best key.
      {
        const int jr = (k + kConsumerWarps - 1) / kConsumerWarps;
        unsigned* pub = sh.pub[i & 1];
        unsigned rem = (m == m) ? float_orderable(m) : 0u;
        for (int r = 0; r < jr; ++r) {
          const unsigned cur = __reduce_max_sync(kFull, rem);
          const unsigned bal = __ballot_sync(kFull, rem == cur);
          if (lane == __ffs(bal) - 1) rem = 0u;
          if (lane == 0) pub[warp * jr + r] = cur;
        }
        consumer_sync();
        const int np = kConsumerWarps * jr;
        const unsigned u = lane < np ? pub[lane] : 0u;
        int gt = 0;
        for (int o = 0; o < np; o += 4) {
          const uint4 v4 = *reinterpret_cast<const uint4*>(pub + o);  // broadcast reads
          gt += (v4.x > u) + (v4.y > u) + (v4.z > u) + (v4.w > u);
        }
        const unsigned vk = __reduce_min_sync(kFull, (lane < np && gt < k) ? u : 0xffffffffu);
        if (vk != 0u && vk != 0xffffffffu) {  // 0: NaN maxima among the top k (row flagged; no bound)
          const unsigned long long b0 = ((unsigned long long)vk << 32) | 0x80000000ull;  // (v_k, INT_MAX)
          if (b0 > bound) bound = b0;
        }
      }
      stamp(P, t0 && i == 0, 5);
      // elements whose value reaches the bound are appended to the warp buffer at positions from
      // a warp prefix sum (no shared atomics); when the buffer would overflow it is compacted to
      // its top-k, the bound tightened and the remaining elements re-filtered
      float bv = bound ? tk_val(bound) : -INFINITY;
      unsigned pend = 0u;
      if (m >= bv) {
#pragma unroll
        for (int n = 0; n < EPT; ++n) pend |= (x[n] >= bv ? 1u : 0u) << n;
      }
      for (;;) {
        const int cnt = __popc(pend);
        int incl, total;
        if (!__any_sync(kFull, cnt > 1)) {  // common case: at most one candidate per lane
          const unsigned bal = __ballot_sync(kFull, cnt > 0);
          incl = __popc(bal & (0xffffffffu >> (31 - lane)));
          total = __popc(bal);
        } else {
          incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
          }
          total = __shfl_sync(kFull, incl, 31);
        }
        if (total == 0) break;
        if (pend) {
          int pos = wcnt + incl - cnt;
          unsigned bits = pend;
          while (bits) {
            const int n = __ffs(bits) - 1;
            bits &= bits - 1u;
            if (pos < kSegBuf) {
              const int idx = elem_index<BF16>(cbase, tid, n);
              float v;
              if (idx >= V) {
                v = -INFINITY;
              } else if (TMA) {  // the stage is still held: reload the element from shared memory
                const char* sp = ring + (size_t)s * kChunkBytes +
                                 ((size_t)((n / EPV) * kConsumers + tid) * EPV + (n % EPV)) * (BF16 ? 2 : 4);
                v = BF16 ? __uint_as_float((uint32_t)(*reinterpret_cast<const unsigned short*>(sp)) << 16)
                         : *reinterpret_cast<const float*>(sp);
              } else {
                const char* rp = row_ptr(P, par, logits, ld_bytes, row, sh.rfe, row0) + (size_t)idx * (BF16 ? 2 : 4);
                v = BF16 ? __uint_as_float((uint32_t)(*reinterpret_cast<const unsigned short*>(rp)) << 16)
                         : *reinterpret_cast<const float*>(rp);
              }
              W.buf[pos] = tk_key(v, idx);
              pend &= ~(1u << n);
            }
            ++pos;
          }
        }
        if (wcnt + total <= kSegBuf) {
          wcnt += total;
          break;
        }
        __syncwarp();
        warp_compact(W, kSegBuf, k, lane);
        wcnt = k;
        if (W.list[k - 1] > bound) bound = W.list[k - 1];
        bv = tk_val(bound);
#pragma unroll
        for (int n = 0; n < EPT; ++n)
          if (!(x[n] >= bv)) pend &= ~(1u << n);
      }
      __syncwarp();
      if (TMA && lane == 0) mbar_arrive(&pipe.empty[s]);  // release the stage
      gstamp(P, t0 && i < 2, 20 + 3 * (int)i);
      stamp(P, t0 && i == 0, 6);
    }
    // ---- segment end: warp buffers (top-k only if longer) -> CTA segment list (rank merge) ----
    if (wcnt > k) {
      warp_compact(W, wcnt, k, lane);
      wcnt = k;
    }
    // padding keys are distinct and below every real key (value -inf, index > INT_MAX)
    if (lane < k) sh.cl[warp * k + lane] = lane < wcnt ? W.buf[lane] : kKeySentinel - 1 - (warp * k + lane);
    wcnt = 0;
    gstamp(P, t0 && q == rr.lo, 24);
    consumer_sync();
    gstamp(P, t0 && q == rr.lo, 28);
    {
      const int n = kConsumerWarps * k;  // even
      if (tid < n) {
        const unsigned long long key = sh.cl[tid];
        const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(sh.cl);
        int r0 = 0, r1 = 0;
#pragma unroll 4
        for (int f = 0; f < n / 2; ++f) {
          const ulonglong2 v = c2[f];
          r0 += (v.x > key);
          r1 += (v.y > key);
        }
        const int rank = r0 + r1;
        if (rank < k) P.segkey[((size_t)row * cpr + c0) * k + rank] = key;
      }
    }
    if (tid == 0) P.seglen[(size_t)row * cpr + c0] = nch;
    gstamp(P, t0 && q == rr.lo, 25);
    consumer_sync();
    // warp 0 alone: arrival (release of the CTA's lists, acquire of the others'), and the row
    // merge when this CTA completed the row; the other warps go on with the next segment
    if (warp == 0) {
      int last = 0;
      if (lane == 0) {
        const int old = atom_add_acq_rel_gpu(&P.row_done[row], nch);  // publish + acquire
        last = (old + nch == cpr);
      }
      last = __shfl_sync(kFull, last, 0);
      gstamp(P, t0 && q == rr.lo, 26);
      if (last) {  // this CTA completed the row
        if (lane == 0) {
          probe_max(P, 3);
          probe_min(P, 8);
        }
        gstamp(P, lane == 0 && row == 0, 29);
        merge_row_warp(P, layer, par, row, mst);
        gstamp(P, lane == 0 && row == 0, 30);
        if (lane == 0) {
          probe_max(P, 4);
          const int old = atom_add_acq_rel_gpu(&P.layer_done[layer - 1], 1);
          if (old + 1 == R) sh.last_layer = 1;
        }
        __syncwarp();
      }
    }
    q += nch;
    ++row;
    c0 = 0;
  }
  if (tid == 0) probe_max(P, 2);
  consumer_sync();
  if (sh.last_layer) {
    if (tid == 0) {
      P.layer_done[layer - 1] = 0;
      probe_max(P, 5);
    }
    if (fuse_select) select_layer<kConsumers>(P, layer, kSelFull, ring);
    if (tid == 0) probe_max(P, 6);
  }
  if (tid == 0) probe_max(P, 7);
  tl_end(P, layer);
}

}  // namespace

size_t layer_smem_bytes(int cpr, int k) {
  return (size_t)kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(ExpandShared) + merge_stage_bytes(cpr, k);
}

int expand_occupancy() {
  int n = 0;
  const int sm = (int)layer_smem_bytes(kMaxCpr, kMaxK);
  cudaFuncSetAttribute(layer_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(layer_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(layer_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(layer_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, layer_kernel<true, true>, kLayerThreads, layer_smem_bytes(16, 10));
  return n > 0 ? n : 1;
}

void launch_expand(const Params& P, int layer, const void* logits, long long ld_bytes, bool tma, bool fuse_select,
                   int grid, cudaStream_t s) {
  const char* base = static_cast<const char*>(logits);
  const size_t smem = layer_smem_bytes(P.cpr, P.k);
  const int f = fuse_select ? 1 : 0;
  if (P.dtype == SMART_BF16) {
    if (tma) launch_k(layer_kernel<true, true>, dim3(grid), dim3(kLayerThreads), smem, s, P, layer, base, ld_bytes, f);
    else launch_k(layer_kernel<true, false>, dim3(grid), dim3(kLayerThreads), smem, s, P, layer, base, ld_bytes, f);
  } else {
    if (tma) launch_k(layer_kernel<false, true>, dim3(grid), dim3(kLayerThreads), smem, s, P, layer, base, ld_bytes, f);
    else launch_k(layer_kernel<false, false>, dim3(grid), dim3(kLayerThreads), smem, s, P, layer, base, ld_bytes, f);
  }
}

}  // namespace smart
