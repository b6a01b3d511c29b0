// mask_verify.cu — begin-step reset, K3 `smart_build_mask` (A7) and K4 `smart_verify_accept` (A8).
//
// A7 ("verifying an entire tree in a single forward pass" needs a tree attention mask):
//   M[i] = M[parent(i)] | bit(i) (ancestor-or-self), pos = root_pos + depth, parent, token.
// A8 (P:453 T = 0; S:383 greedy_match): from the root, t = argmax target(r, cur) (lowest id on
//   ties); follow the child with token t if it exists, else stop with bonus t.  All tree rows'
//   argmaxes are streamed in one HBM pass (same persistent chunk scheduler as K1); the request
//   whose last row completes runs the walk (one warp).
#include "verify_core.cuh"

namespace smart {

__global__ void begin_step_kernel(Params P, const int32_t* root_tok, const int32_t* root_pos) {
  // trigger first: the layer-1 grid (264 clustered CTAs) starts launching while the previous
  // step's tail drains; its griddepcontrol.wait still waits for this kernel's completion
  pdl_trigger();
  pdl_wait();
  tl_start(P, 0);
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < P.b_loc) {
    size_t o = (size_t)r * P.T;
    P.n_nodes[r] = 1;
    P.tok[o] = root_tok ? root_tok[r] : -1;
    P.parent[o] = -1;
    P.depth[o] = 0;
    P.p[o] = 1.f;    // root: p = cum = 1
    P.cum[o] = 1.f;
    P.path_sum[o] = 0.0;
    P.E_r[r] = 0.0;
    P.leaf_cnt[r] = 1;
    P.leaf_sum[r] = 0.0;
    P.finished[r] = 0;
    P.root_pos[r] = root_pos ? root_pos[r] : 0;
    P.fr[0][r] = make_int2(r, 0);  // A_0 = {root}
    P.fr_cum[0][r] = 1.f;
    P.fr_cnt[0][r] = 1;
    P.fr_off[0][r] = r;
  }
  if (blockIdx.x == 0 && threadIdx.x < SMART_MAX_DEPTH) {
    DevTrace t{};
    P.trace[threadIdx.x] = t;
    P.layer_done[threadIdx.x] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x <= SMART_MAX_DEPTH) P.fr_ready[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *P.fr_total[0] = P.b_loc;
    *P.err = 0;
    P.sum_accept[0] = 0ull;
    P.sum_accept[1] = 0ull;
    *P.N_glob = 0;
    *P.E_glob = 0.0;
  }
  tl_end(P, 0);
}

namespace {

// ---- K3: one CTA (1024 threads = 32 warps) for the whole local batch; each warp stages one
// request's (parent, depth, token) arrays in shared memory, then walks ancestors on chip ----
__global__ void __launch_bounds__(1024) mask_kernel(Params P, uint32_t* mask, int32_t* pos, int32_t* parent,
                                                    int32_t* tok, int32_t* tree_len) {
  extern __shared__ int s_tree[];  // [32 warps][3 * T] staged trees, then [b_loc + 1] row offsets
  __shared__ int s_run[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = P.T, MW = P.MW;
  int* s_off = s_tree + 32 * 3 * T;
  tl_start(P, 52);
  pdl_trigger();  // the verify grid may start launching during the last layer (it waits for us)
  pdl_wait();
  tl_start(P, 20);
  int* sp = s_tree + (size_t)warp * 3 * T;
  int* sd = sp + T;
  int* st = sd + T;
  // the warp's first request: its tree is staged while the row-offset scan runs
  int n0 = 0, rp0 = 0;
  if (warp < P.b_loc) {
    const int r = warp;
    n0 = P.n_nodes[r];
    rp0 = P.root_pos[r];
    for (int i = lane; i < n0; i += 32) {
      sp[i] = P.parent[(size_t)r * T + i];
      sd[i] = P.depth[(size_t)r * T + i];
      st[i] = P.tok[(size_t)r * T + i];
    }
  }
  // verify-row offsets: exclusive scan of n_nodes (rows of K4), kept in shared memory too
  {
    const int per = (P.b_loc + 1023) / 1024;
    const int b0 = tid * per, b1 = min(P.b_loc, b0 + per);
    int local = 0;
    for (int r = b0; r < b1; ++r) local += P.n_nodes[r];
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_run[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int v = s_run[lane];
      int iv = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, iv, o);
        if (lane >= o) iv += t;
      }
      s_run[lane] = iv - v;
      if (lane == 31) s_run[32] = iv;
    }
    __syncthreads();
    int run = s_run[warp] + incl - local;
    for (int r = b0; r < b1; ++r) {
      P.vrow_off[r] = run;
      s_off[r] = run;
      run += P.n_nodes[r];
    }
    if (tid == 0) P.vrow_off[P.b_loc] = s_run[32];
    __syncthreads();
  }
  for (int r = warp; r < P.b_loc; r += 32) {
    int n, rp;
    if (r == warp) {  // staged above
      n = n0;
      rp = rp0;
    } else {
      __syncwarp();
      n = P.n_nodes[r];
      rp = P.root_pos[r];
      for (int i = lane; i < n; i += 32) {
        sp[i] = P.parent[(size_t)r * T + i];
        sd[i] = P.depth[(size_t)r * T + i];
        st[i] = P.tok[(size_t)r * T + i];
      }
    }
    const int vo = s_off[r];
    for (int i = lane; i < n; i += 32) P.vrow_rn[vo + i] = make_int2(r, i);  // verify row -> (request, node)
    __syncwarp();
    for (int i = lane; i < T; i += 32) {
      const size_t o = (size_t)r * T + i;
      if (i < n) {
        if (mask) {
          for (int w = 0; w < MW; ++w) {
            uint32_t word = 0;
            for (int j = i; j >= 0; j = sp[j])  // ancestor-or-self chain (depth <= 16)
              if ((j >> 5) == w) word |= 1u << (j & 31);
            mask[o * MW + w] = word;
          }
        }
        if (pos) pos[o] = rp + sd[i];
        if (parent) parent[o] = sp[i];
        if (tok) tok[o] = st[i];
      } else {
        if (mask)
          for (int w = 0; w < MW; ++w) mask[o * MW + w] = 0u;
        if (pos) pos[o] = 0;
        if (parent) parent[o] = -1;
        if (tok) tok[o] = -1;
      }
    }
    if (lane == 0 && tree_len) tree_len[r] = n;
  }
  tl_end(P, 20);
}

struct VerifyShared {
  int2 rn[kStageRows];  // (request, node) of the CTA's first rows
};


// K4: persistent TMA-staged stream over all tree rows (request r, node i < tree_len[r]) of the
// target logits; exact argmax per row (value desc, index asc); the request whose last row
// completes runs the greedy walk.
// the verify stream: 3 stages x 16 KiB per CTA, 3 CTAs per SM (more warps in flight per SM than
// the layer kernel's 2 x 5 stages: the argmax work per element is smaller)
constexpr int kVStages = 3;
using VPipe = StreamPipeT<kVStages>;

// the T > 0 variant at 4 CTAs per SM: it is issue and latency bound (the per-token hash), so more
// resident warps pay more than registers
template <bool BF16, bool TMA, bool SAMPLE>
__global__ void __launch_bounds__(kLayerThreads, SAMPLE ? 4 : 2)
verify_kernel(Params P, const char* __restrict__ target, long long ld_bytes, int32_t* accept_len,
              int32_t* accept_path, int32_t* bonus, float inv_tau, unsigned long long seed) {
  constexpr int EPV = BF16 ? 8 : 4;
  constexpr int ESZ = BF16 ? 2 : 4;
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;
  VPipe& pipe = *reinterpret_cast<VPipe*>(dsm + kVStages * kChunkBytes);
  VerifyShared& sh = *reinterpret_cast<VerifyShared*>(dsm + kVStages * kChunkBytes + sizeof(VPipe));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    mbar_fence_init();
  }
  tl_start(P, 53);
  pdl_wait();
  pdl_trigger();
  tl_start(P, 21);
  const int NR = P.vrow_off[P.b_loc];
  const int cpr = P.cpr, CE = P.chunk_elems, V = P.V, T = P.T;
  const long long row_bytes = (long long)V * ESZ;
  const RowRange rr = cta_range_min(NR * cpr, P.min_units);
  if (rr.lo >= rr.hi) return;
  // the CTA's row descriptors, staged once (no dependent global loads per chunk)
  const int row0 = rr.lo / cpr;
  const int nstage = min((rr.hi - 1) / cpr - row0 + 1, kStageRows);
  if (tid < nstage) sh.rn[tid] = P.vrow_rn[row0 + tid];
  auto rown = [&](int row) { return row - row0 < kStageRows ? sh.rn[row - row0] : P.vrow_rn[row]; };
  auto row_base = [&](int row) {
    const int2 e = rown(row);
    return target + ((long long)e.x * T + e.y) * ld_bytes;
  };
  __syncthreads();
  if (warp == kConsumerWarps) {
    if (TMA && lane == 0) produce(pipe, ring, rr, cpr, row_bytes, row_base);
    return;
  }
  int nanf = 0;
  int i = 0;
  int q = rr.lo;
  int row = row0, c0 = rr.lo - row0 * cpr;
  int seg = -1;
  while (q < rr.hi) {
    ++seg;
    const int nch = min(cpr - c0, rr.hi - q);
    const int2 rnode = rown(row);
    const int r = rnode.x, node = rnode.y;
    const uint32_t rowkey = SAMPLE ? sample_rowkey(seed, (unsigned long long)(P.b_off + r), (unsigned long long)node) : 0u;
    float bv = -INFINITY;
    int bi = kIdxSentinel;
    for (int c = c0; c < c0 + nch; ++c, ++i) {
      gstamp(P, blockIdx.x == 0 && tid == 0 && i < 8, 100 + (int)i);
      const int cbase = c * CE;
      uint4 raw[kVecPerThread];
      if (TMA) {
        const int s = (int)(i % kVStages);
        mbar_wait(&pipe.full[s], (uint32_t)((i / kVStages) & 1));
        const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * kChunkBytes);
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) raw[j] = st[j * kConsumers + tid];
        __syncwarp();
        if (lane == 0) mbar_arrive(&pipe.empty[s]);
      } else {
        const char* rp = row_base(row);
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
          const int e0 = cbase + (j * kConsumers + tid) * EPV;
          uint32_t w[4];
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) w[q2] = BF16 ? 0xff80ff80u : 0xff800000u;
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            if (e0 + e < V) {
              if (BF16) {
                const uint32_t h = *reinterpret_cast<const unsigned short*>(rp + (size_t)(e0 + e) * 2);
                w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0x0000ffffu) | (h << 16)) : ((w[e >> 1] & 0xffff0000u) | h);
              } else {
                w[e] = *reinterpret_cast<const uint32_t*>(rp + (size_t)(e0 + e) * 4);
              }
            }
          raw[j] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      verify_chunk<BF16, SAMPLE>(raw, cbase, V, tid, rowkey, inv_tau, bv, bi, nanf);
    }
    // ---- segment end: every warp posts its best (value desc, index asc) as one 64-bit key with
    // a fire-and-forget red.max on the row's slot; the walk runs in verify_walk_kernel once the
    // grid has completed (no arrivals, merges or barriers here) ----
    if (lane == 0 && bi != kIdxSentinel) {
      const unsigned long long key = ((unsigned long long)vkey_orderable(bv) << 32) | (0xffffffffu - (unsigned)bi);
      asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(P.vbest + (size_t)r * T + node), "l"(key)
                   : "memory");
    }
    gstamp(P, blockIdx.x == 0 && tid == 0 && seg < 4, 110 + 4 * seg + 3);
    q += nch;
    ++row;
    c0 = 0;
  }
  if (nanf) atomicOr(P.err, kErrTargetNaN);
  tl_end(P, 21);
  if (SMART_PROBES && P.dbg && tid == 0) P.dbg[256 + blockIdx.x] = gtime();  // per-CTA end (debug timeline)
}

// A8 walk: one warp per request.  The request's tree (parent, token) is staged in shared
// memory before the dependency wait (the tree is final: the verify grid launched this kernel only
// after its own wait on the mask kernel); after the verify grid completes, the row keys give the
// target argmax of every node; the slots are cleared for the next step.
__global__ void __launch_bounds__(1024) verify_walk_kernel(Params P, int32_t* accept_len, int32_t* accept_path,
                                                           int32_t* bonus) {
  extern __shared__ int s_walk[];  // [32 warps][3 * T]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + warp;
  const int T = P.T;
  int* s_par = s_walk + warp * 3 * T;
  int* s_tok = s_par + T;
  int* s_arg = s_tok + T;
  const int n = r < P.b_loc ? P.n_nodes[r] : 0;
  for (int j = lane; j < n; j += 32) {
    s_par[j] = P.parent[(size_t)r * T + j];
    s_tok[j] = P.tok[(size_t)r * T + j];
  }
  pdl_wait();
  pdl_trigger();
  if (r >= P.b_loc) return;
  for (int j = lane; j < n; j += 32) {
    unsigned long long* slot = P.vbest + (size_t)r * T + j;
    const unsigned long long key = __ldcg(slot);
    s_arg[j] = (int)(0xffffffffu - (uint32_t)key);
    *slot = 0ull;
  }
  __syncwarp();
  const int D = P.d > 0 ? P.d : 1;
  int cur = 0, acc = 0, bon = -1;
  for (;;) {
    const int t = s_arg[cur];
    int found = -1;
    for (int j0 = cur + 1; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool f = j < n && s_par[j] == cur && s_tok[j] == t;
      const unsigned bal = __ballot_sync(kFull, f);
      if (bal) {
        found = j0 + __ffs(bal) - 1;
        break;
      }
    }
    if (found < 0) {
      bon = t;
      break;
    }
    if (lane == 0 && accept_path && acc < D) accept_path[(size_t)r * D + acc] = found;
    ++acc;
    cur = found;
  }
  if (lane == 0) {
    if (accept_len) accept_len[r] = acc;
    if (bonus) bonus[r] = bon;
    atomicAdd(P.sum_accept, (unsigned long long)acc);
    atomicAdd(P.sum_accept + 1, (unsigned long long)(n - 1));
  }
  if (accept_path)
    for (int j = acc + lane; j < D; j += 32) accept_path[(size_t)r * D + j] = -1;
}

}  // namespace

// ---- NEXT #3 stage 2: rerank of the two-stage likelihood-maximising baseline (Q32) ----------
// EAGLE-3 / MSD (Fig. 2(a)(b)): the expansion stage (select_layer in BASELINE mode) kept the
// top-W candidates of every layer by (cum desc, c asc); here every candidate generated in the step
// (admitted or not) competes for the g = floor(B_verify / b) verification slots by (cum desc,
// layer asc, c asc), and the kept set is renumbered in (layer, c) order.  A kept candidate's parent
// has a larger-or-equal cum at a lower layer, so it ranks earlier and is kept too (closure).
// One CTA per request; keys (~bits(cum) << 32 | layer << 16 | c) rank in O(n^2) shared-memory
// counting (n <= d W k candidates).
constexpr int kRerankThreads = 256;

__global__ void __launch_bounds__(kRerankThreads) rerank_kernel(Params P) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int nmax = max(P.d, 1) * P.Wq * P.k;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(sm);
  int* qi = reinterpret_cast<int*>(key + nmax);
  int* fpos = qi + nmax;
  int* newidx = fpos + nmax;
  __shared__ int cnt;
  const int r = blockIdx.x, tid = threadIdx.x;
  pdl_wait();
  pdl_trigger();
  if (tid == 0) cnt = 0;
  for (int i = tid; i < P.T; i += kRerankThreads) newidx[i] = i == 0 ? 0 : -1;
  __syncthreads();
  for (int l = 1; l <= P.d; ++l) {
    const DevTrace& tr = P.trace[l - 1];
    const int R = tr.executed ? tr.n_rows : 0;
    for (int row = tid; row < R; row += kRerankThreads) {
      const int2 rs = __ldcg(&P.cand_rs[(size_t)(l - 1) * P.cap_rows + row]);
      if (rs.x != r) continue;
      const int s = atomicAdd(&cnt, P.k);
      const size_t q0 = (size_t)(l - 1) * P.cap_rows * P.k + (size_t)row * P.k;
      for (int j = 0; j < P.k; ++j) {
        const float c = __ldcg(&P.cand[q0 + j].cum);
        key[s + j] = ((unsigned long long)(~__float_as_uint(c)) << 32) |
                     ((unsigned long long)l << 16) | (unsigned)(rs.y * P.k + j);
        qi[s + j] = (int)(q0 + j);
      }
    }
  }
  __syncthreads();
  const int n = cnt;
  const int keep = min(n, P.B);
  // rank by (cum desc, layer asc, c asc); kept if rank < g
  for (int i = tid; i < n; i += kRerankThreads) {
    const unsigned long long ki = key[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += key[j] < ki;
    fpos[i] = rank < keep ? 0 : -1;
  }
  __syncthreads();
  // final index: 1 + kept candidates before it in (layer, c) order; expanded ones map their node
  for (int i = tid; i < n; i += kRerankThreads) {
    if (fpos[i] < 0) continue;
    const unsigned lo = (unsigned)key[i];
    int pos = 1;
    for (int j = 0; j < n; ++j) pos += (fpos[j] >= 0) && ((unsigned)key[j] < lo);
    fpos[i] = pos;
    const int q = qi[i];
    if (__ldcg(&P.cand_adm[q])) newidx[__ldcg(&P.cand_node[q])] = pos;
  }
  __syncthreads();
  const size_t o = (size_t)r * P.T;
  for (int i = tid; i < n; i += kRerankThreads) {
    const int pos = fpos[i];
    if (pos < 0) continue;
    const Cand cd = P.cand[qi[i]];
    const int par = newidx[cd.parent];
    if (par < 0) atomicExch(P.err, 1);  // closure violated (cannot happen)
    P.tok[o + pos] = cd.tok;
    P.parent[o + pos] = par;
    P.depth[o + pos] = (int)((key[i] >> 16) & 0xffffu);
    P.p[o + pos] = cd.p;
    P.cum[o + pos] = cd.cum;
  }
  if (tid == 0) P.n_nodes[r] = 1 + keep;
}

size_t rerank_smem_bytes(const Params& P) {
  return (size_t)std::max(P.d, 1) * P.Wq * P.k * 16 + (size_t)P.T * 4;
}

cudaError_t rerank_set_smem(size_t bytes) {
  return cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_rerank(const Params& P, cudaStream_t s) {
  launch_k(rerank_kernel, dim3(P.b_loc), dim3(kRerankThreads), rerank_smem_bytes(P), s, P);
}

void launch_mask(const Params& P, uint32_t* mask, int32_t* pos, int32_t* parent, int32_t* tok, int32_t* tree_len,
                 cudaStream_t s) {
  const size_t smem = mask_smem_bytes(P.T, P.b_loc);
  launch_k(mask_kernel, dim3(1), dim3(1024), smem, s, P, mask, pos, parent, tok, tree_len);
}

size_t mask_smem_bytes(int T, int b) { return ((size_t)32 * 3 * T + b + 1) * sizeof(int); }

cudaError_t mask_set_smem_bytes(size_t bytes) {
  // every kernel of the step asks for the maximum shared-memory carveout, so consecutive kernels
  // never wait for an SM's L1/shared split to be reconfigured
  cudaFuncSetAttribute(mask_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(begin_step_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return cudaFuncSetAttribute(mask_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)std::max<size_t>(bytes, 48 * 1024));
}

size_t verify_smem_bytes(int T) {
  (void)T;
  return (size_t)kVStages * kChunkBytes + sizeof(VPipe) + sizeof(VerifyShared);
}

template <bool BF16, bool TMA, bool SAMPLE>
static void verify_attr(int sm) {
  cudaFuncSetAttribute(verify_kernel<BF16, TMA, SAMPLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(verify_kernel<BF16, TMA, SAMPLE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
}

int verify_occupancy(bool sample) {
  int n = 0;
  const int sm = (int)verify_smem_bytes(1024);
  verify_attr<true, true, false>(sm);
  verify_attr<true, false, false>(sm);
  verify_attr<false, true, false>(sm);
  verify_attr<false, false, false>(sm);
  verify_attr<true, true, true>(sm);
  verify_attr<true, false, true>(sm);
  verify_attr<false, true, true>(sm);
  verify_attr<false, false, true>(sm);
  // the T > 0 kernel holds more registers: its own occupancy sizes its grid (no second wave)
  if (sample)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, verify_kernel<true, true, true>, kLayerThreads,
                                                  verify_smem_bytes(1024));
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, verify_kernel<true, true, false>, kLayerThreads,
                                                  verify_smem_bytes(1024));
  return n > 0 ? n : 1;
}

template <bool SAMPLE>
static void launch_verify_t(const Params& P, const char* t, long long ld_bytes, bool tma, int32_t* accept_len,
                            int32_t* accept_path, int32_t* bonus, int grid, cudaStream_t s, float inv_tau,
                            unsigned long long seed) {
  const size_t sm = verify_smem_bytes(P.T);
  const dim3 g(grid), blk(kLayerThreads);
  if (P.dtype == SMART_BF16) {
    if (tma) launch_k(verify_kernel<true, true, SAMPLE>, g, blk, sm, s, P, t, ld_bytes, accept_len, accept_path, bonus, inv_tau, seed);
    else launch_k(verify_kernel<true, false, SAMPLE>, g, blk, sm, s, P, t, ld_bytes, accept_len, accept_path, bonus, inv_tau, seed);
  } else {
    if (tma) launch_k(verify_kernel<false, true, SAMPLE>, g, blk, sm, s, P, t, ld_bytes, accept_len, accept_path, bonus, inv_tau, seed);
    else launch_k(verify_kernel<false, false, SAMPLE>, g, blk, sm, s, P, t, ld_bytes, accept_len, accept_path, bonus, inv_tau, seed);
  }
}

void launch_verify(const Params& P, const void* target, long long ld_bytes, bool tma, int32_t* accept_len,
                   int32_t* accept_path, int32_t* bonus, int grid, cudaStream_t s, bool sample, float inv_tau,
                   unsigned long long seed) {
  const char* t = static_cast<const char*>(target);
  if (sample) launch_verify_t<true>(P, t, ld_bytes, tma, accept_len, accept_path, bonus, grid, s, inv_tau, seed);
  else launch_verify_t<false>(P, t, ld_bytes, tma, accept_len, accept_path, bonus, grid, s, inv_tau, seed);
  launch_k(verify_walk_kernel, dim3((P.b_loc + 31) / 32), dim3(1024), walk_smem_bytes(P.T), s, P, accept_len,
           accept_path, bonus);
}

size_t walk_smem_bytes(int T) { return (size_t)32 * 3 * T * sizeof(int); }

cudaError_t walk_set_smem_bytes(size_t bytes) {
  cudaFuncSetAttribute(verify_walk_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  return cudaFuncSetAttribute(verify_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)std::max<size_t>(bytes, 48 * 1024));
}

}  // namespace smart
