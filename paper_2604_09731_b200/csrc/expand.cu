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

// logits row of frontier row `row` (layer parity `par`)
__device__ __forceinline__ const char* row_ptr(const Params& P, int par, const char* base, long long ld_bytes,
                                              int row) {
  if (P.row_mode == SMART_ROWS_NODE) {
    const int2 fe = P.fr[par][row];
    return base + ((long long)fe.x * P.T + fe.y) * ld_bytes;
  }
  return base + (long long)row * ld_bytes;
}

// per-warp top-k state in shared memory (64-bit keys)
struct WarpTopk {
  unsigned long long buf[kSegBuf];  // candidates of the current segment (appended; compacted)
  unsigned long long list[kMaxK];   // compacted top-k, sorted best first
  int cnt;
};

struct ExpandShared {
  unsigned long long tau;  // CTA threshold hint (best k-th key bound of any warp)
  int last, last_layer;
  WarpTopk w[kConsumerWarps];
  float red[kConsumerWarps];
  int2 fe;
  float pc;
  int nseg;
};

// row-merge staging, carved from the dynamic shared memory after ExpandShared (sized by cpr, k)
struct MergeStage {
  float2* ms;                // [cpr * 8] softmax partials
  unsigned long long* keys;  // [cpr * k] segment lists
  int* seglen;               // [cpr]
  int* segstart;             // [cpr] chunk index of each existing segment
};

__host__ __device__ inline size_t merge_stage_bytes(int cpr, int k) {
  return (size_t)cpr * kConsumerWarps * 8 + (size_t)cpr * k * 8 + (size_t)cpr * 8 + 16;
}

__device__ inline MergeStage merge_stage(char* base, int cpr, int k) {
  MergeStage m;
  m.ms = reinterpret_cast<float2*>(base);
  m.keys = reinterpret_cast<unsigned long long*>(m.ms + cpr * kConsumerWarps);
  m.seglen = reinterpret_cast<int*>(m.keys + cpr * k);
  m.segstart = m.seglen + cpr;
  return m;
}

// Warp-level compaction: list <- top-k of buf[0..n) by rank counting (keys distinct, except
// sentinels which never rank inside the top-k of a buffer holding >= k real keys); the buffer
// then restarts from the list.
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
  if (lane == 0) w.cnt = min(n, k);
  __syncwarp();
}

// ---- row merge by the CTA that completed the row (256 consumer threads) ----
// Everything the merge needs is fetched in one wave into shared memory, then merged by rank.
__device__ void merge_row(const Params& P, int layer, int par, int row, ExpandShared& sh, MergeStage st) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = P.k, cpr = P.cpr;
  const int npart = cpr * kConsumerWarps;
  const float2* ms = P.ms + (size_t)row * npart;
  for (int q = tid; q < npart; q += kConsumers) st.ms[q] = __ldcg(&ms[q]);
  for (int c = tid; c < cpr; c += kConsumers) {
    st.seglen[c] = __ldcg(&P.seglen[(size_t)row * cpr + c]);
    P.seglen[(size_t)row * cpr + c] = 0;  // self-cleaning for the next use
  }
  for (int q = tid; q < cpr * k; q += kConsumers) st.keys[q] = __ldcg(&P.segkey[(size_t)row * cpr * k + q]);
  if (tid == 0) {
    const int2 fe = P.fr[par][row];
    sh.fe = fe;
    sh.pc = P.cum[(size_t)fe.x * P.T + fe.y];
    sh.nseg = 0;
  }
  consumer_sync();
  for (int c = tid; c < cpr; c += kConsumers)
    if (st.seglen[c] > 0) st.segstart[atomicAdd(&sh.nseg, 1)] = c;
  // (1) softmax normaliser: M = max, Z = sum s*exp(m - M), association fixed by cpr only
  float m = -INFINITY;
  for (int q = tid; q < npart; q += kConsumers) m = fmaxf(m, st.ms[q].x);
  m = warp_max(m);
  if (lane == 0) sh.red[warp] = m;
  consumer_sync();
  float M = sh.red[0];
#pragma unroll
  for (int w = 1; w < kConsumerWarps; ++w) M = fmaxf(M, sh.red[w]);
  const float ML = M * kLog2e;
  float z = 0.f;
  for (int q = tid; q < npart; q += kConsumers) {
    const float2 v = st.ms[q];
    if (v.y != 0.f || isnan(v.y)) z += v.y * ex2(fmaf(v.x, kLog2e, -ML));
  }
  z = warp_sum(z);
  consumer_sync();  // everyone has read sh.red (M); segstart complete
  if (lane == 0) sh.red[warp] = z;
  consumer_sync();
  float Z = 0.f;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) Z += sh.red[w];
  // (2) exact top-k of the union of the existing segment lists, by rank
  const int nseg = sh.nseg;
  const int n = nseg * k;
  const int2 fe = sh.fe;
  const float pc = sh.pc;
  for (int e = tid; e < n; e += kConsumers) {
    const int es = e / k;  // once per entry (not in the inner loop)
    const unsigned long long key = st.keys[st.segstart[es] * k + (e - es * k)];
    int rank = 0;
    for (int s2 = 0; s2 < nseg; ++s2) {
      const unsigned long long* Lk = st.keys + st.segstart[s2] * k;
#pragma unroll 8
      for (int f = 0; f < k; ++f) rank += (Lk[f] > key);
    }
    if (rank < k) {
      // (3) A1 probability and A2 path score of the rank-th candidate
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
  if (tid == 0) {
    P.cand_rs[(size_t)(layer - 1) * P.cap_rows + row] = make_int2(fe.x, row - P.fr_off[par][fe.x]);
    P.rowstat[row] = make_float2(M, Z);
    if (!(Z >= 1.0f) || isinf(Z) || isnan(M)) atomicOr(P.err, kErrDraftNaN);  // Q23
    P.row_done[row] = 0;
  }
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
    probe_min(P, 0);
    probe_max(P, 1);
  }
  const int R = *P.fr_total[par];
  if (R == 0) {
    // A_{l-1} is empty for every request: the step has terminated at this layer
    if (fuse_select && blockIdx.x == 0 && tid == 0) *P.fr_total[layer & 1] = 0;
    return;
  }
  const int k = P.k, cpr = P.cpr, CE = P.chunk_elems, V = P.V;
  const long long row_bytes = (long long)V * (BF16 ? 2 : 4);
  const RowRange rr = cta_range_min((long long)R * cpr, P.min_units);
  if (rr.lo >= rr.hi) return;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    mbar_fence_init();
    sh.tau = 0ull;
    sh.last_layer = 0;
  }
  if (tid < kConsumerWarps) sh.w[tid].cnt = 0;
  __syncthreads();

  if (warp == kConsumerWarps) {  // ---- producer warp ----
    if (TMA && lane == 0)
      produce(pipe, ring, rr, cpr, row_bytes, [&](int row) { return row_ptr(P, par, logits, ld_bytes, row); });
    return;
  }

  // ---- consumer warps ----
  WarpTopk& W = sh.w[warp];
  long long i = 0;
  long long q = rr.lo;
  while (q < rr.hi) {
    const int row = (int)(q / cpr);
    const int c0 = (int)(q % cpr);
    const int nch = (int)min((long long)(cpr - c0), rr.hi - q);
    unsigned long long bound = 0ull;  // lower bound of the segment's k-th best key
    for (int c = c0; c < c0 + nch; ++c, ++i) {
      uint4 raw[kVecPerThread];
      if (TMA) {
        const int s = (int)(i % kStages);
        mbar_wait(&pipe.full[s], (uint32_t)((i / kStages) & 1));
        const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * kChunkBytes);
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) raw[j] = st[j * kConsumers + tid];
        __syncwarp();
        if (lane == 0) mbar_arrive(&pipe.empty[s]);  // release the stage as soon as it is in registers
      } else {
        load_direct<BF16>(row_ptr(P, par, logits, ld_bytes, row), c * CE, V, tid, raw);
      }
      float x[EPT];
      unpack<BF16>(raw, x);
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
      const float Mw = warp_max(m);
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      if (Mw != -INFINITY) {
        const float ML = Mw * kLog2e;
#pragma unroll
        for (int n = 0; n < EPT; ++n) s4[n & 3] += ex2(fmaf(x[n], kLog2e, -ML));
      }
      const float sacc = warp_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
      if (lane == 0) P.ms[((size_t)row * cpr + c) * kConsumerWarps + warp] = make_float2(Mw, sacc);

      // ---- top-k candidates of this warp-chunk ----
      if (c == c0) {
        // segment seeding: v_k = k-th largest lane-maximum VALUE; k distinct elements have
        // value >= v_k, so key(v_k, INT_MAX) is a valid lower bound of the k-th best key
        const unsigned om = (m == m) ? float_orderable(m) : 0u;
        unsigned thr = 0xffffffffu, vk = 0u;
        int got = 0;
        for (int it = 0; it < k && got < k; ++it) {
          const unsigned cur = __reduce_max_sync(kFull, om < thr ? om : 0u);
          got += __popc(__ballot_sync(kFull, om == cur));
          thr = cur;
          vk = cur;
        }
        if (got >= k) {
          const unsigned long long b0 = ((unsigned long long)vk << 32) | 0x80000000ull;  // (v_k, INT_MAX)
          if (b0 > bound) bound = b0;
        }
      }
      {
        const unsigned long long hk = *(volatile unsigned long long*)&sh.tau;
        if (hk > bound) bound = hk;
      }
      if (W.cnt > kSegBuf - 32) {  // keep room for this chunk's appends
        warp_compact(W, W.cnt, k, lane);
        if (W.list[k - 1] > bound) bound = W.list[k - 1];
      }
      const float bv = tk_val(bound);
      bool cl = (m >= bv) && (m == m);
      unsigned pushed = 0u;
      while (__any_sync(kFull, cl)) {
        bool more = false;
        if (cl) {
#pragma unroll
          for (int j = 0; j < kVecPerThread; ++j)
            if (vm[j] >= bv) {
#pragma unroll
              for (int e = 0; e < EPV; ++e) {
                const int n = j * EPV + e;
                if (x[n] >= bv && !((pushed >> n) & 1u)) {
                  const unsigned long long key = tk_key(x[n], elem_index<BF16>(cbase, tid, n));
                  if (key >= bound) {
                    const int slot = atomicAdd(&W.cnt, 1);
                    if (slot < kSegBuf) {
                      W.buf[slot] = key;
                      pushed |= 1u << n;
                    } else {
                      more = true;
                    }
                  }
                }
              }
            }
        }
        __syncwarp();
        cl = more;
        if (__any_sync(kFull, more)) {  // buffer full: compact, tighten, retry the rest
          if (lane == 0) W.cnt = kSegBuf;
          __syncwarp();
          warp_compact(W, kSegBuf, k, lane);
          if (W.list[k - 1] > bound) bound = W.list[k - 1];
        }
      }
      if (lane == 0 && bound) atomicMax(&sh.tau, bound);
    }
    // ---- segment end: warp buffers -> warp top-k -> CTA segment list (rank merge), arrival ----
    warp_compact(W, W.cnt, k, lane);
    if (lane == 0) W.cnt = 0;
    consumer_sync();
    for (int t = tid; t < kConsumerWarps * k; t += kConsumers) {  // only the 8k live entries
      const int tw = t / k, te = t - tw * k;
      const unsigned long long key = sh.w[tw].list[te];
      int rank = 0;
      for (int w = 0; w < kConsumerWarps; ++w) {
#pragma unroll 8
        for (int f = 0; f < k; ++f) rank += (sh.w[w].list[f] > key);
      }
      if (rank < k) P.segkey[((size_t)row * cpr + c0) * k + rank] = key;
    }
    if (tid == 0) P.seglen[(size_t)row * cpr + c0] = nch;
    consumer_sync();
    if (tid == 0) {
      const int old = atom_add_acq_rel_gpu(&P.row_done[row], nch);  // publish + acquire
      sh.last = (old + nch == cpr);
      sh.tau = 0ull;
    }
    consumer_sync();
    if (sh.last) {
      if (tid == 0) {
        probe_max(P, 3);
        probe_min(P, 8);
      }
      merge_row(P, layer, par, row, sh, mst);
      if (tid == 0) probe_max(P, 4);
      consumer_sync();
      if (tid == 0) {
        const int old = atom_add_acq_rel_gpu(&P.layer_done[layer - 1], 1);
        sh.last_layer = (old + 1 == R);
      }
      consumer_sync();
    }
    q += nch;
  }
  if (tid == 0) probe_max(P, 2);
  if (sh.last_layer) {
    if (tid == 0) {
      P.layer_done[layer - 1] = 0;
      probe_max(P, 5);
    }
    if (fuse_select) select_layer<kConsumers>(P, layer, kSelFull, ring);
    if (tid == 0) probe_max(P, 6);
  }
  if (tid == 0) probe_max(P, 7);
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
    if (tma) layer_kernel<true, true><<<grid, kLayerThreads, smem, s>>>(P, layer, base, ld_bytes, f);
    else layer_kernel<true, false><<<grid, kLayerThreads, smem, s>>>(P, layer, base, ld_bytes, f);
  } else {
    if (tma) layer_kernel<false, true><<<grid, kLayerThreads, smem, s>>>(P, layer, base, ld_bytes, f);
    else layer_kernel<false, false><<<grid, kLayerThreads, smem, s>>>(P, layer, base, ld_bytes, f);
  }
}

}  // namespace smart
