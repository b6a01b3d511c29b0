// expand.cu — the per-layer kernel: K1 `smart_expand_step` (A1 top-k + softmax of every frontier
// row; A2 path score cum = cum(parent) * p, Eq.(3)) with the
// layer's selection A3-A6 fused into the tail of the last CTA (single rank).
//
// Design:
//  * Row teams in thread-block clusters: the persistent grid is made of 8-CTA clusters; from the
//    layer's row count R each cluster is cut into teams of t in {8,4,2,1} CTAs (the largest t
//    with R <= #teams, t <= chunks per row), and team n streams rows n, n + #teams, ...  Each
//    member CTA takes a balanced slice of every row's 16 KiB chunks; its partial results go
//    straight into the team leader's shared memory (DSMEM stores + one remote mbarrier arrive),
//    and a dedicated merge warp in the leader finishes the row: no global round trip between
//    the stream and the row result.
//  * HBM stream, TMA-staged: per CTA a producer warp bulk-copies chunks (cp.async.bulk +
//    mbarrier tx count) into a 6-stage shared-memory ring; 8 consumer warps read 16-byte
//    vectors from it.
//  * softmax: each consumer warp reduces its 1024 (bf16) / 512 (fp32) elements of a chunk to
//    (max, sum exp) with a fixed shuffle tree; the CTA that streamed a chunk combines its 8 warp
//    partials in warp order, and the row merge combines the cpr chunk partials in fixed order, so
//    Z is bit-identical for any grid size, team layout or sharding.
//  * top-k (exact, ties -> lower index): keys are 64-bit (orderable value | ~index), so one
//    compare orders two candidates.  Per warp and segment (consecutive chunks of one row in one
//    CTA) a running lower bound of the k-th best key is kept: at the segment's first chunk it is
//    the k-th largest lane-maximum value (k rounds of a one-instruction warp max), later tightened
//    by compactions and a CTA-wide hint.  Only the 16-byte vectors whose max reaches the bound
//    are scanned; qualifying elements are appended to a per-warp buffer in shared memory, which
//    is compacted to its top-k (rank counting) when full and at the segment end.
//  * the leader's merge warp computes Z (association fixed by the chunk count), the exact top-k
//    of the members' lists (threshold + rank), p and cum; the CTA whose merge warp completes the
//    layer's last row (one acq_rel arrival per row) runs the selection (select_core.cuh).
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

// per-warp top-k state in shared memory (64-bit keys)
struct WarpTopk {
  unsigned long long buf[kSegBuf];  // candidates of the current row slice (appended; compacted)
  unsigned long long list[kMaxK];   // compacted top-k, sorted best first
};

constexpr int kCluster = 8;                          // CTAs per cluster (portable maximum)
constexpr int kMergeWarp = kConsumerWarps + 1;       // warp 9: row merges in team leaders
constexpr int kLayerThreadsT = kLayerThreads + 32;   // 320 threads: consumers, producer, merger

struct __align__(16) ExpandShared {
  unsigned long long tau;                         // slice-wide bound: max over warps of their k-th best
  int2 rfe[kStageRows];                           // frontier entries of the team's rows
  float rcum[kStageRows];                         // their path scores (cum of the parent node)
  __align__(16) unsigned pub[2][kConsumerWarps * kMaxK];        // slice start: top-k lane maxima per warp
  __align__(16) unsigned long long cl[kConsumerWarps * kMaxK];  // slice end: each warp's top-k
  uint64_t ready[2];  // leader: all members' partials of the team's n-th row are in (parity n & 1)
  uint64_t freeb[2];  // every CTA: the leader has consumed buffer parity p (remote arrive)
  WarpTopk w[kConsumerWarps];
};

// team buffers, carved after ExpandShared.  Receive side (the team leader's copy, double-
// buffered by row parity): softmax partials [cpr][8 warps] and lists [kCluster][kp].  Send side
// (every CTA): its slice's partials and top-k list, staged locally and moved to the leader with
// one shared::cluster bulk copy each (completion counted on the leader's mbarrier).
// kp = k rounded up to even, so every bulk copy is a multiple of 16 bytes.
__host__ __device__ inline int list_stride(int k) { return (k + 1) & ~1; }

struct TeamBuf {
  float4* ms[2];              // receive: per-chunk softmax partials (M_c, S_c, -, -) [cpr]
  unsigned long long* lists[2];
  unsigned long long* surv;  // merge scratch [kCluster * kp]
  float2* msl;               // this CTA's (chunk, warp) partials [cpr][8]
  unsigned long long* listl; // send staging: this CTA's top-k [kp]
  float4* msc;               // send staging: this CTA's per-chunk partials [cpr]
};

__host__ __device__ inline size_t team_buf_bytes(int cpr, int k) {
  const size_t kp = (size_t)list_stride(k);
  return 2 * ((size_t)cpr * 16 + (size_t)kCluster * kp * 8) + (size_t)kCluster * kp * 8 +
         (size_t)cpr * kConsumerWarps * 8 + kp * 8 + (size_t)cpr * 16;
}

__device__ inline TeamBuf team_buf(char* base, int cpr, int k) {
  const int kp = list_stride(k);
  TeamBuf t;
  char* p = base;
  for (int b = 0; b < 2; ++b) {
    t.ms[b] = reinterpret_cast<float4*>(p);
    p += (size_t)cpr * 16;
    t.lists[b] = reinterpret_cast<unsigned long long*>(p);
    p += (size_t)kCluster * kp * 8;
  }
  t.surv = reinterpret_cast<unsigned long long*>(p);
  p += (size_t)kCluster * kp * 8;
  t.msl = reinterpret_cast<float2*>(p);
  p += (size_t)cpr * kConsumerWarps * 8;
  t.listl = reinterpret_cast<unsigned long long*>(p);
  p += (size_t)kp * 8;
  t.msc = reinterpret_cast<float4*>(p);
  return t;
}

// ---- cluster / DSMEM primitives ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {  // local smem -> cluster address
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t a, uint32_t count) {  // remote, release.cluster
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)  // suspend-time hint: sleep instead of re-polling (each poll invalidates L1)
      : "memory");
}
// bulk copy of `bytes` (multiple of 16) from this CTA's shared memory to a cluster address,
// completion (tx bytes) signalled on the destination CTA's mbarrier
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "r"(smem_u32(src)), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// ---- row merge by the team leader's merge warp, from its own shared memory ----
// M = max, Z = sum s*exp(m - M) over the row's cpr x 8 partials (association fixed by cpr);
// T = the best k-th entry over the members' lists (each list is its slice's top-k, so T bounds the
// row's k-th best key from below); the entries >= T are ranked among themselves and the top k
// written with p (A1) and cum (A2, Eq.(3)).
__device__ void merge_row_team(const Params& P, int layer, int par, int row, int2 fe, float pc, int slot, int t,
                               const float4* ms, const unsigned long long* lists, unsigned long long* surv,
                               bool pr) {
  const int lane = threadIdx.x & 31;
  const int k = P.k, cpr = P.cpr;
  stamp(P, pr, 1);
  // (1) softmax normaliser from the cpr per-chunk partials (each already combined over its 8
  // warps in fixed order by the member that streamed the chunk): M = max, Z = sum S_c exp(M_c - M)
  // in a fixed association (lane-strided, then the xor tree) -- a function of cpr only
  // (cpr <= 64: at most two partials per lane, loaded once; the sum stays lane-strided in order)
  const float4 v0 = lane < cpr ? ms[lane] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const float4 v1 = lane + 32 < cpr ? ms[lane + 32] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  const float M = warp_max_fast(fmaxf(v0.x, v1.x));
  const float ML = M * kLog2e;
  float z = 0.f;
  z += (v0.y != 0.f || isnan(v0.y)) ? v0.y * ex2(fmaf(v0.x, kLog2e, -ML)) : 0.f;
  z += (v1.y != 0.f || isnan(v1.y)) ? v1.y * ex2(fmaf(v1.x, kLog2e, -ML)) : 0.f;
  const float Z = warp_sum(z);
  const float rZ = __frcp_rn(Z);  // correctly rounded 1/Z (no division slow path)
  stamp(P, pr, 2);
  // (2) threshold: best tail over the members' lists
  const int kp = list_stride(k);
  const unsigned long long tail = lane < t ? lists[lane * kp + k - 1] : 0ull;
  const unsigned th = __reduce_max_sync(kFull, (unsigned)(tail >> 32));
  const unsigned tl = __reduce_max_sync(kFull, (unsigned)(tail >> 32) == th ? (unsigned)tail : 0u);
  const unsigned long long T = ((unsigned long long)th << 32) | tl;
  // (3) survivors, compacted by ballot
  const int nkey = t * kp;  // the padding slot of an odd k holds a key below every real one
  int ns = 0;
  for (int e0 = 0; e0 < nkey; e0 += 32) {
    const int e = e0 + lane;
    const unsigned long long key = e < nkey ? lists[e] : 0ull;
    const bool sv = e < nkey && key >= T;
    const unsigned bal = __ballot_sync(kFull, sv);
    if (sv) surv[ns + __popc(bal & ((1u << lane) - 1u))] = key;
    ns += __popc(bal);
  }
  __syncwarp();
  stamp(P, pr, 3);
  // (4) exact top-k among the survivors; A1 p and A2 cum
  auto emit = [&](unsigned long long key, int rank) {
    const float v = tk_val(key);
    const float pj = ex2(fmaf(v, kLog2e, -ML)) * rZ;  // p = exp(x - M) / Z   (tau = 1, Q10)
    Cand cd;
    cd.tok = tk_idx(key);
    cd.p = pj;
    cd.cum = pc * pj;  // Eq.(3)
    cd.parent = fe.y;
    P.cand[((size_t)(layer - 1) * P.cap_rows + row) * k + rank] = cd;
  };
  if (ns <= 32) {
    // one survivor per lane; rank by broadcast compares (no shared-memory loop)
    const unsigned long long mine = lane < ns ? surv[lane] : 0ull;
    int rank = 0;
#pragma unroll 8
    for (int q = 0; q < ns; ++q) rank += (__shfl_sync(kFull, mine, q) > mine);
    if (lane < ns && rank < k) emit(mine, rank);
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
      if (rank < k) emit(key, rank);
    }
  }
  stamp(P, pr, 4);
  if (lane == 0) {
    P.cand_rs[(size_t)(layer - 1) * P.cap_rows + row] = make_int2(fe.x, slot);
    if (!(Z >= 1.0f) || isinf(Z) || isnan(M)) atomicOr(P.err, kErrDraftNaN);  // Q23
  }
  __syncwarp();
}

template <bool BF16, bool TMA>
__global__ void __launch_bounds__(kLayerThreadsT, 2)
layer_kernel(Params P, int layer, const char* __restrict__ logits, long long ld_bytes, int flags) {
  // flags bit 0: the layer's selection is fused (the grid's last cluster); bit 1: early start —
  // the previous layer's selection was fused and publishes its frontier with a release flag
  // (P.fr_ready[layer - 1]) before its kernel ends, so streaming CTAs wait on that flag instead of
  // the previous grid's completion (the select CTA still waits for the completion: it reads the
  // per-request state the previous selection writes after the frontier)
  const int fuse_select = flags & 1;
  const bool early = (flags & 2) != 0;
  constexpr int EPT = Traits<BF16>::EPT;
  constexpr int EPV = Traits<BF16>::EPV;
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;
  StreamPipe& pipe = *reinterpret_cast<StreamPipe*>(dsm + kStages * kChunkBytes);
  ExpandShared& sh = *reinterpret_cast<ExpandShared*>(dsm + kStages * kChunkBytes + sizeof(StreamPipe));
  const TeamBuf tb = team_buf(dsm + kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(ExpandShared), P.cpr, P.k);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1;
  const uint32_t crank = cluster_ctarank();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    mbar_init(&sh.ready[0], 1);  // the leader's arrive.expect_tx; members complete the bytes
    mbar_init(&sh.ready[1], 1);
    mbar_init(&sh.freeb[0], 1);
    mbar_init(&sh.freeb[1], 1);
    mbar_fence_init();
    sh.tau = 0ull;
  }
  cluster_sync_all();  // barriers initialised cluster-wide before any remote arrive
  tl_start(P, 32 + layer);
#if SMART_PROBES
  if (SMART_PROBES && P.dbg && tid == 0 && blockIdx.x < 384) P.dbg[256 + blockIdx.x] = gtime();  // per-CTA start
#endif
  const bool sel_cta0 = fuse_select && (int)blockIdx.x == (int)gridDim.x - kCluster;
  if (!early || sel_cta0) pdl_wait();
  pdl_trigger();
  if (early && !sel_cta0) {
    if (tid == 0) wait_flag(&P.fr_ready[layer - 1], P.err);
    __syncthreads();
  }
  tl_start(P, layer);
  // the first row's frontier entry for each possible team size t = 8 >> tid, fetched together
  // with the row count (the team layout is only known once R is)
  int2 sfe = make_int2(0, 0);
  float scum = 0.f;
  if (tid < 4) {
    const int row = (int)blockIdx.x / (kCluster >> tid);
    if (row < P.cap_rows) {
      sfe = __ldcg(&P.fr[par][row]);
      scum = __ldcg(&P.fr_cum[par][row]);
    }
  }
  const int R = __ldcg(P.fr_total[par]);
  const bool t0 = (blockIdx.x == 0 && tid == 0);
  gstamp(P, t0, 16);
  if (R == 0) {
    // A_{l-1} is empty for every request: the step has terminated at this layer
    if (fuse_select && blockIdx.x == 0 && tid == 0) {
      *P.fr_total[layer & 1] = 0;
      publish_flag(&P.fr_ready[layer]);
    }
    return;  // no remote traffic in this launch: early exit is safe
  }
  const int k = P.k, cpr = P.cpr, CE = P.chunk_elems, V = P.V;
  const long long row_bytes = (long long)V * (BF16 ? 2 : 4);
  // ---- team layout from R: largest t in {8,4,2,1} with R <= #teams and t <= cpr ----
  // with the fused selection the grid's last cluster is reserved: its rank-0 CTA runs A3-A6
  const int S = fuse_select ? (int)gridDim.x - kCluster : (int)gridDim.x;
  const bool sel_cta = fuse_select && (int)blockIdx.x == S;
  // (t is a power of two: shifts, no integer division in the prologue)
  int lt = 3;  // log2 t
  while (lt > 0 && (R > (S >> lt) || (1 << lt) > cpr)) --lt;
  const int t = 1 << lt;
  const int nteams = S >> lt;
  const int team = (int)blockIdx.x >> lt, member = (int)blockIdx.x & (t - 1);
  const uint32_t lrank = crank - (uint32_t)member;  // the team leader's rank in the cluster
  const int nrows = ((int)blockIdx.x < S && team < R)
                        ? ((nteams & (nteams - 1)) == 0 ? (R - team + nteams - 1) >> (31 - __clz(nteams))
                                                        : (R - team + nteams - 1) / nteams)
                        : 0;
  const int mlo = (member * cpr) >> lt, mhi = ((member + 1) * cpr) >> lt;  // this CTA's chunks of each row
  const int nstage = min(nrows, kStageRows);
  const int tsel = (t == 8) ? 0 : (t == 4) ? 1 : (t == 2) ? 2 : 3;
  if (nstage > 0 && tid == tsel) {
    sh.rfe[0] = sfe;
    sh.rcum[0] = scum;
  }
  if (tid >= 4 && tid - 3 < nstage) {  // further rows (large layers)
    const int n = tid - 3;
    const int row = team + n * nteams;
    sh.rfe[n] = __ldcg(&P.fr[par][row]);
    sh.rcum[n] = __ldcg(&P.fr_cum[par][row]);
  }
  __syncthreads();
  gstamp(P, t0, 17);
  auto rowfe = [&](int n, int row) { return n < kStageRows ? sh.rfe[n] : __ldcg(&P.fr[par][row]); };
  auto rowp = [&](int n, int row) -> const char* {
    if (P.row_mode == SMART_ROWS_NODE) {
      const int2 fe = rowfe(n, row);
      return logits + ((long long)fe.x * P.T + fe.y) * ld_bytes;
    }
    if (P.row_mode == SMART_ROWS_POSITION) {  // DFLASH: the request's position-l row
      const int2 fe = rowfe(n, row);
      return logits + ((long long)fe.x * P.d + (layer - 1)) * ld_bytes;
    }
    return logits + (long long)row * ld_bytes;
  };

  if (warp == kConsumerWarps) {
    // ---- producer warp: the member's chunks of each of the team's rows, in order ----
    if (TMA && lane == 0) {
      int i = 0;
      for (int n = 0; n < nrows; ++n) {
        const int row = team + n * nteams;
        const char* base = rowp(n, row);
        for (int c = mlo; c < mhi; ++c, ++i) {
          const int s = i % kStages;
          mbar_wait(&pipe.empty[s], ((uint32_t)(i / kStages) & 1u) ^ 1u);
          const long long off = (long long)c * kChunkBytes;
          const uint32_t bytes = (uint32_t)min((long long)kChunkBytes, row_bytes - off);
          mbar_expect_tx(&pipe.full[s], bytes);
          bulk_g2s(ring + (size_t)s * kChunkBytes, base + off, bytes, &pipe.full[s]);
        }
      }
    }
  } else if (warp == kMergeWarp) {
    // ---- merge warp (team leaders): finish each of the team's rows once all members are in ----
    if (member == 0) {
      for (int n = 0; n < nrows; ++n) {
        const int row = team + n * nteams;
        const int b = n & 1;
        const int2 fe = rowfe(n, row);
        const float pc = n < kStageRows ? sh.rcum[n] : __ldcg(&P.fr_cum[par][row]);
        const int slot = row - __ldcg(&P.fr_off[par][fe.x]);  // frontier slot within the request (loaded while waiting)
        if (lane == 0)  // this row's bytes: all chunk partials + t lists
          mbar_expect_tx(&sh.ready[b], (uint32_t)(cpr * 16 + t * list_stride(k) * 8));
        mbar_wait_acq_cluster(&sh.ready[b], (uint32_t)(n >> 1) & 1u);
        gstamp(P, blockIdx.x == 0 && lane == 0 && n == 0, 24);
        merge_row_team(P, layer, par, row, fe, pc, slot, t, tb.ms[b], tb.lists[b], tb.surv,
                       blockIdx.x == 0 && lane == 0 && n == 0);
        stamp(P, blockIdx.x == 0 && lane == 0 && n == 0, 5);
        gstamp(P, blockIdx.x == 0 && lane == 0 && n == 0, 25);
        // buffer b is free again (only awaited when the team streams another row into it)
        if (lane < t && n + 2 < nrows) mbar_arrive_cluster(mapa_rank(&sh.freeb[b], lrank + lane), 1);
        if (lane == 0) {
          red_add_release_gpu(&P.layer_done[layer - 1], 1);  // row done (the select CTA polls)
          stamp(P, blockIdx.x == 0 && n == 0, 6);
          gstamp(P, blockIdx.x == 0 && n == 0, 26);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- consumer warps ----
    WarpTopk& W = sh.w[warp];
    int wcnt = 0;  // entries in W.buf (warp-uniform)
    int i = 0;
    for (int n = 0; n < nrows; ++n) {
      const int row = team + n * nteams;
      const int b = n & 1;
      if (n >= 2) mbar_wait_acq_cluster(&sh.freeb[b], (uint32_t)((n - 2) >> 1) & 1u);  // leader done with b
      if (n >= 1) {  // the previous slice's bulk copies have read the send staging
        if (tid == 0) bulk_wait_read();
        consumer_sync();
      }
      unsigned long long bound = 0ull;  // lower bound of the slice's k-th best key
      for (int c = mlo; c < mhi; ++c, ++i) {
        uint4 raw[kVecPerThread];
        const int s = i % kStages;
        if (TMA) {
          mbar_wait(&pipe.full[s], ((uint32_t)(i / kStages)) & 1u);
          gstamp(P, t0 && i < 2, 18 + 3 * i);
          const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * kChunkBytes);
#pragma unroll
          for (int j = 0; j < kVecPerThread; ++j) raw[j] = st[j * kConsumers + tid];
        } else {
          load_direct<BF16>(rowp(n, row), c * CE, V, tid, raw);
        }
        if (P.debug_mode == 1) {  // timing experiment: stream only
          __syncwarp();
          if (TMA && lane == 0) mbar_arrive(&pipe.empty[s]);
          continue;
        }
        float x[EPT];
        unpack<BF16>(raw, x);
        const int cbase = c * CE;
        if (c == cpr - 1) {  // ragged last chunk: elements past the row end -> -inf
#pragma unroll
          for (int e = 0; e < EPT; ++e)
            if (elem_index<BF16>(cbase, tid, e) >= V) x[e] = -INFINITY;
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
        const float Mw = warp_max_fast(m);
        // exp2(x*log2e - M*log2e) on element pairs: FFMA2 + 2 MUFU + FADD2 (two pair accumulators)
        unsigned long long acc2[2] = {0ull, 0ull};
        if (Mw != -INFINITY && P.debug_mode != 4) {  // (debug_mode 4: timing experiment, no exps)
          const float ML = Mw * kLog2e;
          const unsigned long long l2e2 = f2pk(kLog2e, kLog2e), nml2 = f2pk(-ML, -ML);
#pragma unroll
          for (int e = 0; e < EPT; e += 2) {
            const unsigned long long y = ffma2(f2pk(x[e], x[e + 1]), l2e2, nml2);
            acc2[(e >> 1) & 1] = fadd2(acc2[(e >> 1) & 1], f2pk(ex2(f2lo(y)), ex2(f2hi(y))));
          }
        }
        const float sacc = warp_sum((f2lo(acc2[0]) + f2hi(acc2[0])) + (f2lo(acc2[1]) + f2hi(acc2[1])));
        gstamp(P, t0 && i < 2, 19 + 3 * i);
        if (lane == 0) tb.msl[(c - mlo) * kConsumerWarps + warp] = make_float2(Mw, sacc);
        if (P.debug_mode == 3) {  // timing experiment only: softmax without the top-k filter
          __syncwarp();
          if (TMA && lane == 0) mbar_arrive(&pipe.empty[s]);
          continue;
        }

        const bool pq = t0 && i < 2;  // probe: CTA 0, warp 0 lane 0, first two chunks
        stamp(P, pq, 24 + 4 * i);
        // ---- top-k candidates of this warp-chunk ----
        // CTA-wide bound at the slice's first chunk: every warp publishes its top-j lane maxima
        // (j = ceil(k/8), one lane per round, so ties keep their multiplicity); these 8j values
        // are distinct elements of the row, so their k-th largest v_k bounds the row's k-th best
        // value from below and key(v_k, INT_MAX) bounds the slice's k-th best key.  Later chunks
        // run barrier-free on the warp's own bound (tightened by compaction).
        if (c == mlo) {
          // every warp publishes its top-j lane maxima (j >= 2 rounds of a warp max; ties keep
          // their multiplicity); v_k, the k-th largest of these 8j values, bounds the slice's
          // k-th best value from below
          const int jr = max((k + kConsumerWarps - 1) / kConsumerWarps, 2);
          unsigned* pub = sh.pub[i & 1];
          unsigned rem = (m == m) ? float_orderable(m) : 0u;
          for (int r = 0; r < jr; ++r) {
            const unsigned cur = __reduce_max_sync(kFull, rem);
            const unsigned bal = __ballot_sync(kFull, rem == cur);
            if (lane == __ffs(bal) - 1) rem = 0u;
            if (lane == 0) pub[warp * jr + r] = cur;
          }
          consumer_sync();
          const int np = kConsumerWarps * jr;  // multiple of 8
          unsigned vc = 0xffffffffu;
          for (int e = lane; e < np; e += 32) {
            const unsigned u = pub[e];
            int gt = 0;
            for (int o = 0; o < np; o += 4) {
              const uint4 v4 = *reinterpret_cast<const uint4*>(pub + o);  // broadcast reads
              gt += (v4.x > u) + (v4.y > u) + (v4.z > u) + (v4.w > u);
            }
            if (gt < k && u < vc) vc = u;
          }
          const unsigned vk = __reduce_min_sync(kFull, vc);
          if (vk != 0u && vk != 0xffffffffu) {  // 0: NaN maxima among the top k (row flagged; no bound)
            const unsigned long long b0 = ((unsigned long long)vk << 32) | 0x80000000ull;  // (v_k, INT_MAX)
            if (b0 > bound) bound = b0;
          }
        }
        // elements whose value reaches the bound are appended to the warp buffer at positions from
        // a warp prefix sum (no shared atomics); when the buffer would overflow it is compacted to
        // its top-k, the bound tightened and the remaining elements re-filtered
        stamp(P, pq && i == 0, 31);
        {
          // barrier-free CTA bound: every warp posts its k-th best after each compaction (a lower
          // bound of the slice's k-th best) with a shared atomic max; all warps adopt the maximum
          const unsigned long long tt = *reinterpret_cast<volatile unsigned long long*>(&sh.tau);
          if (tt > bound) bound = tt;
        }
        float bv = bound ? tk_val(bound) : -INFINITY;
        if (__any_sync(kFull, m >= bv)) {  // most chunks of a long slice have no candidate at all
          // vectors whose max reaches the bound are expanded cooperatively: each group of EPV
          // lanes takes one such vector (its elements re-read from the still-held ring stage),
          // compares them with the bound and appends the survivors at ballot-prefix positions
          constexpr int G = 32 / EPV;  // vectors per pass
          stamp(P, pq, 25 + 4 * i);
#pragma unroll
          for (int j = 0; j < kVecPerThread; ++j) {
            unsigned bal = __ballot_sync(kFull, vm[j] >= bv);
            while (bal) {
              if (wcnt > kSegBuf - 32) {  // keep room for a full pass: compact, tighten, re-filter
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
                  const char* sp = TMA ? ring + (size_t)s * kChunkBytes +
                                             ((size_t)(j * kConsumers + tl) * EPV + (e % EPV)) * (BF16 ? 2 : 4)
                                       : rowp(n, row) + (size_t)idx * (BF16 ? 2 : 4);
                  v = BF16 ? __uint_as_float((uint32_t)(*reinterpret_cast<const unsigned short*>(sp)) << 16)
                           : *reinterpret_cast<const float*>(sp);
                }
                q = v >= bv;  // NaN never qualifies (the row merge flags it)
              }
              const unsigned qb = __ballot_sync(kFull, q);
              if (q) W.buf[wcnt + __popc(qb & ((1u << lane) - 1u))] = tk_key(v, idx);
              wcnt += __popc(qb);
            }
          }
        }
        stamp(P, pq, 26 + 4 * i);
        if (wcnt >= 2 * k && c + 1 < mhi) {  // keep the warp's buffer short
          __syncwarp();
          warp_compact(W, wcnt, k, lane);
          wcnt = k;
          if (W.list[k - 1] > bound) bound = W.list[k - 1];
          if (lane == 0) atomicMax(&sh.tau, W.list[k - 1]);
        }
        __syncwarp();
        stamp(P, pq && i == 0, 27);
        if (TMA && lane == 0) mbar_arrive(&pipe.empty[s]);  // release the stage
        gstamp(P, t0 && i < 2, 20 + 3 * i);
      }
      // ---- slice end: warp buffers (top-k only if longer) -> CTA list (rank merge) -> leader ----
      if (wcnt > k) {
        warp_compact(W, wcnt, k, lane);
        wcnt = k;
      }
      // padding keys are distinct and below every real key (value -inf, index > INT_MAX)
      if (lane < k) sh.cl[warp * k + lane] = lane < wcnt ? W.buf[lane] : kKeySentinel - 1 - (warp * k + lane);
      wcnt = 0;
      consumer_sync();
      gstamp(P, t0 && n == 0, 31);
      {
        // rank of each of the nl = 8k entries against the whole list (broadcast 16-byte reads:
        // one shared-memory wavefront per load)
        const int nl = kConsumerWarps * k;  // even
        if (tid < nl) {
          const unsigned long long key = sh.cl[tid];
          const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(sh.cl);
          int r0 = 0, r1 = 0;
#pragma unroll 4
          for (int f = 0; f < nl / 2; ++f) {
            const ulonglong2 v = c2[f];
            r0 += (v.x > key);
            r1 += (v.y > key);
          }
          const int rank = r0 + r1;
          if (rank < k) tb.listl[rank] = key;
        }
        if ((k & 1) && tid == 0) tb.listl[k] = kKeySentinel - 1000;  // even-k padding slot
        // per-chunk softmax partials: the 8 warps' (M_w, s_w) of each of this CTA's chunks
        // combined in warp order (fixed association: a function of the chunk alone)
        for (int cc = kConsumers - 1 - tid; cc < mhi - mlo; cc += kConsumers) {
          const float2* pw = tb.msl + cc * kConsumerWarps;
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
          tb.msc[cc] = make_float4(Mc, Sc, 0.f, 0.f);
        }
      }
      gstamp(P, t0 && n == 0, 96);
      consumer_sync();  // staging complete
      gstamp(P, t0 && n == 0, 97);
      if (tid == 0) {
        // two bulk copies into the leader's buffers; their bytes complete its ready barrier
        fence_proxy_async_smem();
        const uint32_t bar = mapa_rank(&sh.ready[b], lrank);
        const int kp = list_stride(k);
        bulk_s2cluster(mapa_rank(tb.ms[b] + mlo, lrank), tb.msc, (uint32_t)((mhi - mlo) * 16), bar);
        bulk_s2cluster(mapa_rank(tb.lists[b] + member * kp, lrank), tb.listl, (uint32_t)(kp * 8), bar);
        bulk_commit();
        gstamp(P, t0 && n == 0, 98);
        sh.tau = 0ull;  // next slice (other warps read it only after the next slice's first barrier)
      }
      gstamp(P, t0 && n == 0, 27);
    }
  }
  if (sel_cta && warp < kConsumerWarps) {
    // ---- the layer's selection: prefetch + A3 now, then wait for the R row merges ----
    gstamp(P, tid == 0, 28);
    const int* done = &P.layer_done[layer - 1];
    int pass = 0;
    auto wait_rows = [&]() {
      if (tid == 0 && pass == 0) {
        while (ld_acquire_gpu(done) < R) {
        }
        P.layer_done[layer - 1] = 0;  // no further arrivals this launch
      }
      consumer_sync();
      gstamp(P, tid == 0, 30);
    };
    // (P.debug_mode == 2: timing experiment only, a second pass through the same code)
    const int npass = P.debug_mode == 2 ? 2 : 1;
    for (; pass < npass; ++pass) {
      if (pass) consumer_sync();
      select_layer<kConsumers>(P, layer, kSelFull, ring, wait_rows);
    }
    gstamp(P, tid == 0, 29);
  }
  if (tid == 0) bulk_wait_read();  // staging buffers stay valid until the copies have read them
#if SMART_PROBES
  if (SMART_PROBES && P.dbg && tid == 0 && blockIdx.x < 384) P.dbg[640 + blockIdx.x] = gtime();  // per-CTA work end
#endif
  // every CTA stays until the cluster is done with its shared memory (remote stores / arrives)
  cluster_sync_all();
  tl_end(P, layer);
}

}  // namespace

size_t layer_smem_bytes(int cpr, int k) {
  return (size_t)kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(ExpandShared) + team_buf_bytes(cpr, k);
}

// grid of the layer kernel: all co-resident 8-CTA clusters (persistent)
int expand_grid(int cpr, int k) {
  const size_t sm = layer_smem_bytes(cpr, k);
  const size_t smax = layer_smem_bytes(kMaxCpr, kMaxK);
  cudaFuncSetAttribute(layer_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  cudaFuncSetAttribute(layer_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  cudaFuncSetAttribute(layer_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  cudaFuncSetAttribute(layer_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
  cudaFuncSetAttribute(layer_kernel<true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(layer_kernel<true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(layer_kernel<false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(layer_kernel<false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCluster * 64);
  cfg.blockDim = dim3(kLayerThreadsT);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, layer_kernel<true, true>, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    ncl = 1;
  }
  return ncl * kCluster;
}

void launch_expand(const Params& P, int layer, const void* logits, long long ld_bytes, bool tma, bool fuse_select,
                   bool early, int grid, cudaStream_t s) {
  const char* base = static_cast<const char*>(logits);
  const size_t smem = layer_smem_bytes(P.cpr, P.k);
  const int f = (fuse_select ? 1 : 0) | (early && pdl_enabled() ? 2 : 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kLayerThreadsT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (P.dtype == SMART_BF16) {
    if (tma) cudaLaunchKernelEx(&cfg, layer_kernel<true, true>, P, layer, base, ld_bytes, f);
    else cudaLaunchKernelEx(&cfg, layer_kernel<true, false>, P, layer, base, ld_bytes, f);
  } else {
    if (tma) cudaLaunchKernelEx(&cfg, layer_kernel<false, true>, P, layer, base, ld_bytes, f);
    else cudaLaunchKernelEx(&cfg, layer_kernel<false, false>, P, layer, base, ld_bytes, f);
  }
}

}  // namespace smart
