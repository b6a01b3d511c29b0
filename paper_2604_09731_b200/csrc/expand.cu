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
#include "expand_core.cuh"
#include "select_core.cuh"

namespace smart {

namespace {

constexpr int kCluster = 8;                          // CTAs per cluster (portable maximum)
constexpr int kMergeWarp = kConsumerWarps + 1;       // warp 9: row merges in team leaders
constexpr int kLayerThreadsT = kLayerThreads + 32;   // 320 threads: consumers, producer, merger

struct __align__(16) ExpandShared {
  ConsShared cs;                                  // consumer state (expand_core.cuh)
  int2 rfe[kStageRows];                           // frontier entries of the team's rows
  float rcum[kStageRows];                         // their path scores (cum of the parent node)
  uint64_t ready[2];  // leader: all members' partials of the team's n-th row are in (parity n & 1)
  uint64_t freeb[2];  // every CTA: the leader has consumed buffer parity p (remote arrive)
};

// team buffers, carved after ExpandShared.  Receive side (the team leader's copy, double-
// buffered by row parity): softmax partials [cpr][8 warps] and lists [kCluster][kp].  Send side
// (every CTA): its slice's partials and top-k list, staged locally and moved to the leader with
// one shared::cluster bulk copy each (completion counted on the leader's mbarrier).
// kp = k rounded up to even, so every bulk copy is a multiple of 16 bytes.

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

// ---- row merge by the team leader's merge warp, from its own shared memory (merge_row in
// expand_core.cuh): Z from the cpr per-chunk partials, T = best tail over the t member lists, the
// survivors ranked; A1 p and A2 cum (Eq.(3)) written as the row's k candidate records ----
__device__ void merge_row_team(const Params& P, int layer, int row, int2 fe, float pc, int slot, int t,
                               const float4* ms, const unsigned long long* lists, unsigned long long* surv) {
  const int lane = threadIdx.x & 31;
  const int k = P.k;
  Cand* out = P.cand + ((size_t)(layer - 1) * P.cap_rows + row) * k;
  const bool ok = merge_row(
      k, P.cpr, t, pc, [&](int c) { return ms[c]; }, [&](int e) { return lists[e]; }, surv,
      [&](int rank, int tok, float p, float cum) {
        Cand cd;
        cd.tok = tok;
        cd.p = p;
        cd.cum = cum;
        cd.parent = fe.y;
        out[rank] = cd;
      });
  if (lane == 0) {
    P.cand_rs[(size_t)(layer - 1) * P.cap_rows + row] = make_int2(fe.x, slot);
    if (!ok) atomicOr(P.err, kErrDraftNaN);  // Q23
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
    sh.cs.tau = 0ull;
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
        merge_row_team(P, layer, row, fe, pc, slot, t, tb.ms[b], tb.lists[b], tb.surv);
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
    // ---- consumer warps (expand_core.cuh) ----
    int wcnt = 0;  // entries in the warp's buffer (warp-uniform)
    float wrun = -INFINITY;  // the warp's running max over the current slice
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
        const char* stage = ring + (size_t)s * kChunkBytes;
        if (TMA) {
          mbar_wait(&pipe.full[s], ((uint32_t)(i / kStages)) & 1u);
          gstamp(P, t0 && i < 2, 18 + 3 * i);
          const uint4* st = reinterpret_cast<const uint4*>(stage);
#pragma unroll
          for (int j = 0; j < kVecPerThread; ++j) raw[j] = st[j * kConsumers + tid];
        } else {
          load_direct<BF16>(rowp(n, row), c * CE, V, tid, raw);
        }
        consume_chunk<BF16, TMA>(P, sh.cs, tb.msl, raw, stage, TMA ? nullptr : rowp(n, row), c, mlo, mhi, i, wcnt,
                                 bound, wrun);
        __syncwarp();
        if (TMA && lane == 0) mbar_arrive(&pipe.empty[s]);  // release the stage
        gstamp(P, t0 && i < 2, 20 + 3 * i);
      }
      // ---- slice end: warp buffers -> CTA list (rank merge) -> leader ----
      slice_end_post(sh.cs, k, wcnt);
      gstamp(P, t0 && n == 0, 31);
      slice_end_merge(
          sh.cs, tb.msl, k, mhi - mlo, [&](int rank, unsigned long long key) { tb.listl[rank] = key; },
          [&](int cc, float Mc, float Sc) { tb.msc[cc] = make_float4(Mc, Sc, 0.f, 0.f); });
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
        sh.cs.tau = 0ull;  // next slice (other warps read it only after the next slice's first barrier)
      }
      gstamp(P, t0 && n == 0, 27);
    }
  }
  if (sel_cta && warp < kConsumerWarps) {
    // ---- the layer's selection: prefetch + A3 now, then wait for the R row merges ----
    gstamp(P, tid == 0, 28);
    const int* done = &P.layer_done[layer - 1];
    int pass = 0;
    auto wait_rows = [&](SelLayout&, int4*) {
      if (tid == 0 && pass == 0) {
        while (ld_acquire_gpu(done) < R) {
        }
        P.layer_done[layer - 1] = 0;  // no further arrivals this launch
      }
      consumer_sync();
      gstamp(P, tid == 0, 30);
      return false;
    };
    // (P.debug_mode == 2: timing experiment only, a second pass through the same code)
    const int npass = P.debug_mode == 2 ? 2 : 1;
    for (; pass < npass; ++pass) {
      if (pass) consumer_sync();
      select_layer<kConsumers>(P, layer, kSelFull, ring, wait_rows, PubReady{&P.fr_ready[layer]});
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
