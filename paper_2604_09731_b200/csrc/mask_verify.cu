// mask_verify.cu — begin-step reset, K3 `smart_build_mask` (A7) and K4 `smart_verify_accept` (A8).
//
// A7 ("verifying an entire tree in a single forward pass" needs a tree attention mask):
//   M[i] = M[parent(i)] | bit(i) (ancestor-or-self), pos = root_pos + depth, parent, token.
// A8 (P:453 T = 0; S:383 greedy_match): from the root, t = argmax target(r, cur) (lowest id on
//   ties); follow the child with token t if it exists, else stop with bonus t.  All tree rows'
//   argmaxes are streamed in one HBM pass (same persistent chunk scheduler as K1); the request
//   whose last row completes runs the walk (one warp).
#include "stream.cuh"

namespace smart {

namespace {

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

}  // namespace

__global__ void begin_step_kernel(Params P, const int32_t* root_tok, const int32_t* root_pos) {
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
    P.fr_cnt[0][r] = 1;
    P.fr_off[0][r] = r;
  }
  if (blockIdx.x == 0 && threadIdx.x < SMART_MAX_DEPTH) {
    DevTrace t{};
    P.trace[threadIdx.x] = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *P.fr_total[0] = P.b_loc;
    *P.err = 0;
    *P.sum_accept = 0ull;
    *P.N_glob = 0;
    *P.E_glob = 0.0;
  }
}

namespace {

// ---- K3: one CTA (1024 threads = 32 warps) for the whole local batch; each warp stages one
// request's (parent, depth, token) arrays in shared memory, then walks ancestors on chip ----
__global__ void __launch_bounds__(1024) mask_kernel(Params P, uint32_t* mask, int32_t* pos, int32_t* parent,
                                                    int32_t* tok, int32_t* tree_len) {
  extern __shared__ int s_tree[];  // [32 warps][3 * T]
  __shared__ int s_run[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = P.T, MW = P.MW;
  // verify-row offsets: exclusive scan of n_nodes (rows of K4)
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
      run += P.n_nodes[r];
    }
    if (tid == 0) P.vrow_off[P.b_loc] = s_run[32];
  }
  int* sp = s_tree + (size_t)warp * 3 * T;
  int* sd = sp + T;
  int* st = sd + T;
  for (int r = warp; r < P.b_loc; r += 32) {
    const int n = P.n_nodes[r];
    const int rp = P.root_pos[r];
    for (int i = lane; i < n; i += 32) {
      sp[i] = P.parent[(size_t)r * T + i];
      sd[i] = P.depth[(size_t)r * T + i];
      st[i] = P.tok[(size_t)r * T + i];
    }
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
    __syncwarp();
  }
}

struct VerifyShared {
  float wv[kConsumerWarps];
  int wi[kConsumerWarps];
  int last, rlast;
  int walk[1];  // [3 * T] staged (parent, token, argmax) of the walked request (dynamic tail)
};

__device__ __forceinline__ int find_request(const Params& P, int row) {
  int a = 0, b = P.b_loc - 1;
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (P.vrow_off[m] <= row) a = m;
    else b = m - 1;
  }
  return a;
}

// K4: persistent TMA-staged stream over all tree rows (request r, node i < tree_len[r]) of the
// target logits; exact argmax per row (value desc, index asc); the request whose last row
// completes runs the greedy walk.
template <bool BF16, bool TMA>
__global__ void __launch_bounds__(kLayerThreads, 2)
verify_kernel(Params P, const char* __restrict__ target, long long ld_bytes, int32_t* accept_len,
              int32_t* accept_path, int32_t* bonus) {
  constexpr int EPV = BF16 ? 8 : 4;
  constexpr int ESZ = BF16 ? 2 : 4;
  constexpr int EPT = kVecPerThread * EPV;
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;
  StreamPipe& pipe = *reinterpret_cast<StreamPipe*>(dsm + kStages * kChunkBytes);
  VerifyShared& sh = *reinterpret_cast<VerifyShared*>(dsm + kStages * kChunkBytes + sizeof(StreamPipe));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NR = P.vrow_off[P.b_loc];
  const int cpr = P.cpr, CE = P.chunk_elems, V = P.V, T = P.T;
  const long long row_bytes = (long long)V * ESZ;
  const RowRange rr = cta_range_min((long long)NR * cpr, P.min_units);
  if (rr.lo >= rr.hi) return;
  auto row_base = [&](int row) {
    const int r = find_request(P, row);
    return target + ((long long)r * T + (row - P.vrow_off[r])) * ld_bytes;
  };
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kConsumerWarps) {
    if (TMA && lane == 0) produce(pipe, ring, rr, cpr, row_bytes, row_base);
    return;
  }
  int nanf = 0;
  long long i = 0;
  long long q = rr.lo;
  while (q < rr.hi) {
    const int row = (int)(q / cpr);
    const int c0 = (int)(q % cpr);
    const int nch = (int)min((long long)(cpr - c0), rr.hi - q);
    const int r = find_request(P, row);
    const int node = row - P.vrow_off[r];
    float bv = -INFINITY;
    int bi = kIdxSentinel;
    for (int c = c0; c < c0 + nch; ++c, ++i) {
      const int cbase = c * CE;
      float x[EPT];
      if (TMA) {
        const int s = (int)(i % kStages);
        mbar_wait(&pipe.full[s], (uint32_t)((i / kStages) & 1));
        const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * kChunkBytes);
        uint4 raw[kVecPerThread];
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) raw[j] = st[j * kConsumers + tid];
        __syncwarp();
        if (lane == 0) mbar_arrive(&pipe.empty[s]);
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
          const uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            if (BF16) {
              x[j * 8 + 2 * q2] = __uint_as_float(w[q2] << 16);
              x[j * 8 + 2 * q2 + 1] = __uint_as_float(w[q2] & 0xffff0000u);
            } else {
              x[j * 4 + q2] = __uint_as_float(w[q2]);
            }
          }
        }
        if (c == cpr - 1) {
#pragma unroll
          for (int n = 0; n < EPT; ++n)
            if (cbase + ((n / EPV) * kConsumers + tid) * EPV + (n % EPV) >= V) x[n] = -INFINITY;
        }
      } else {
        const char* rp = row_base(row);
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
          const int e0 = cbase + (j * kConsumers + tid) * EPV;
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            float xv = -INFINITY;
            if (e0 + e < V) {
              if (BF16) xv = __uint_as_float(((uint32_t)*reinterpret_cast<const unsigned short*>(rp + (size_t)(e0 + e) * 2)) << 16);
              else xv = *reinterpret_cast<const float*>(rp + (size_t)(e0 + e) * 4);
            }
            x[j * EPV + e] = xv;
          }
        }
      }
      float m = -INFINITY;
#pragma unroll
      for (int n = 0; n < EPT; ++n) m = fmax_nan(m, x[n]);
      if (m != m) nanf = 1;
      int mi = kIdxSentinel;
#pragma unroll
      for (int n = 0; n < EPT; ++n) {
        const int gi = cbase + ((n / EPV) * kConsumers + tid) * EPV + (n % EPV);
        if (x[n] == m && mi == kIdxSentinel && gi < V) mi = gi;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(kFull, m, o);
        const int oi = __shfl_xor_sync(kFull, mi, o);
        if (better(ov, oi, m, mi)) {
          m = ov;
          mi = oi;
        }
      }
      if (better(m, mi, bv, bi)) {
        bv = m;
        bi = mi;
      }
    }
    if (lane == 0) {
      sh.wv[warp] = bv;
      sh.wi[warp] = bi;
    }
    consumer_sync();
    if (tid == 0) {
      float v = sh.wv[0];
      int ix = sh.wi[0];
      for (int w = 1; w < kConsumerWarps; ++w)
        if (better(sh.wv[w], sh.wi[w], v, ix)) {
          v = sh.wv[w];
          ix = sh.wi[w];
        }
      const size_t so = (size_t)row * cpr + c0;
      P.vsegv[so] = v;
      P.vsegi[so] = ix;
      P.vseglen[so] = nch;
      __threadfence();
      const int old = atomicAdd(&P.row_done[row], nch);
      sh.last = (old + nch == cpr);
    }
    consumer_sync();
    if (sh.last && warp == 0) {
      __threadfence();
      float v = -INFINITY;
      int ix = kIdxSentinel;
      for (int c = lane; c < cpr; c += 32) {
        const size_t so = (size_t)row * cpr + c;
        if (__ldcg(&P.vseglen[so]) > 0) {
          const float sv = __ldcg(&P.vsegv[so]);
          const int si = __ldcg(&P.vsegi[so]);
          if (better(sv, si, v, ix)) {
            v = sv;
            ix = si;
          }
          P.vseglen[so] = 0;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(kFull, v, o);
        const int oi = __shfl_xor_sync(kFull, ix, o);
        if (better(ov, oi, v, ix)) {
          v = ov;
          ix = oi;
        }
      }
      int rl = 0;
      if (lane == 0) {
        P.vrow_arg[(size_t)r * T + node] = ix;
        P.row_done[row] = 0;
        __threadfence();
        const int old = atomicAdd(&P.req_done[r], 1);
        rl = (old + 1 == P.n_nodes[r]);
      }
      rl = __shfl_sync(kFull, rl, 0);
      if (rl) {
        // greedy walk of request r: follow the child whose token is the target argmax.
        // The request's tree (parent, token, row argmax) is staged in shared memory first.
        __threadfence();
        const int n = P.n_nodes[r];
        const int D = P.d > 0 ? P.d : 1;
        int* s_par = sh.walk;
        int* s_tok = sh.walk + T;
        int* s_arg = sh.walk + 2 * T;
        for (int j = lane; j < n; j += 32) {
          s_par[j] = P.parent[(size_t)r * T + j];
          s_tok[j] = P.tok[(size_t)r * T + j];
          s_arg[j] = __ldcg(&P.vrow_arg[(size_t)r * T + j]);
        }
        __syncwarp();
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
          P.req_done[r] = 0;
        }
        if (accept_path)
          for (int j = acc + lane; j < D; j += 32) accept_path[(size_t)r * D + j] = -1;
      }
    }
    consumer_sync();
    q += nch;
  }
  if (nanf) atomicOr(P.err, kErrTargetNaN);
}

}  // namespace

void launch_mask(const Params& P, uint32_t* mask, int32_t* pos, int32_t* parent, int32_t* tok, int32_t* tree_len,
                 cudaStream_t s) {
  const size_t smem = (size_t)32 * 3 * P.T * sizeof(int);
  mask_kernel<<<1, 1024, smem, s>>>(P, mask, pos, parent, tok, tree_len);
}

cudaError_t mask_set_smem() {
  return cudaFuncSetAttribute(mask_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 3 * 1024 * 4);
}

size_t verify_smem_bytes(int T) {
  return (size_t)kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(VerifyShared) + (size_t)3 * T * 4;
}

int verify_occupancy() {
  int n = 0;
  const int sm = (int)verify_smem_bytes(1024);
  cudaFuncSetAttribute(verify_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(verify_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(verify_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(verify_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, verify_kernel<true, true>, kLayerThreads, verify_smem_bytes(1024));
  return n > 0 ? n : 1;
}

void launch_verify(const Params& P, const void* target, long long ld_bytes, bool tma, int32_t* accept_len,
                   int32_t* accept_path, int32_t* bonus, int grid, cudaStream_t s) {
  const char* t = static_cast<const char*>(target);
  const size_t sm = verify_smem_bytes(P.T);
  if (P.dtype == SMART_BF16) {
    if (tma) verify_kernel<true, true><<<grid, kLayerThreads, sm, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
    else verify_kernel<true, false><<<grid, kLayerThreads, sm, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
  } else {
    if (tma) verify_kernel<false, true><<<grid, kLayerThreads, sm, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
    else verify_kernel<false, false><<<grid, kLayerThreads, sm, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
  }
}

}  // namespace smart
