// mask_verify.cu — begin-step reset, K3 `smart_build_mask` (A7) and K4 `smart_verify_accept` (A8).
//
// A7 ("verifying an entire tree in a single forward pass" needs a tree attention mask):
//   M[i] = M[parent(i)] | bit(i) (ancestor-or-self), pos = root_pos + depth, parent, token.
// A8 (P:453 T = 0; S:383 greedy_match): from the root, t = argmax target(r, cur) (lowest id on
//   ties); follow the child with token t if it exists, else stop with bonus t.  All tree rows'
//   argmaxes are streamed in one HBM pass (same persistent chunk scheduler as K1); the request
//   whose last row completes runs the walk (one warp).
#include "smart_internal.cuh"

namespace smart {

namespace {

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
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

// ---- K3: one CTA (1024 threads) for the whole local batch ----
__global__ void __launch_bounds__(1024) mask_kernel(Params P, uint32_t* mask, int32_t* pos, int32_t* parent,
                                                    int32_t* tok, int32_t* tree_len) {
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
      int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_run[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int v = s_run[lane], iv = v;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(kFull, iv, o);
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
  const int total = P.b_loc * T;
  for (int idx = tid; idx < total; idx += 1024) {
    const int r = idx / T, i = idx % T;
    const int n = P.n_nodes[r];
    const size_t o = (size_t)r * T + i;
    if (i < n) {
      if (mask) {
        for (int w = 0; w < MW; ++w) {
          uint32_t word = 0;
          for (int j = i; j >= 0; j = P.parent[(size_t)r * T + j])
            if ((j >> 5) == w) word |= 1u << (j & 31);
          mask[o * MW + w] = word;
        }
      }
      if (pos) pos[o] = P.root_pos[r] + P.depth[o];
      if (parent) parent[o] = P.parent[o];
      if (tok) tok[o] = P.tok[o];
    } else {
      if (mask)
        for (int w = 0; w < MW; ++w) mask[o * MW + w] = 0u;
      if (pos) pos[o] = 0;
      if (parent) parent[o] = -1;
      if (tok) tok[o] = -1;
    }
    if (i == 0 && tree_len) tree_len[r] = n;
  }
}

struct VerifyShared {
  float wv[kStreamWarps];
  int wi[kStreamWarps];
  int last, rlast;
  float bv;
  int bi;
};

template <bool BF16, bool ALIGNED>
__global__ void __launch_bounds__(kStreamThreads, 2)
verify_kernel(Params P, const char* __restrict__ target, long long ld_bytes, int32_t* accept_len,
              int32_t* accept_path, int32_t* bonus) {
  constexpr int EPV = BF16 ? 8 : 4;
  constexpr int ESZ = BF16 ? 2 : 4;
  constexpr int EPT = kVecPerThread * EPV;
  __shared__ VerifyShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NR = P.vrow_off[P.b_loc];
  const int cpr = P.cpr, CE = P.chunk_elems, V = P.V, T = P.T;
  const long long TOT = (long long)NR * cpr;
  const long long lo = TOT * blockIdx.x / gridDim.x;
  const long long hi = TOT * (blockIdx.x + 1) / gridDim.x;
  int nanf = 0;
  long long q = lo;
  while (q < hi) {
    const int row = (int)(q / cpr);
    const int c0 = (int)(q % cpr);
    const int nch = (int)min((long long)(cpr - c0), hi - q);
    // row -> (request, node) by binary search over vrow_off
    int a = 0, b = P.b_loc - 1;
    while (a < b) {
      int m = (a + b + 1) >> 1;
      if (P.vrow_off[m] <= row) a = m;
      else b = m - 1;
    }
    const int r = a, i = row - P.vrow_off[a];
    const char* rp = target + ((long long)r * T + i) * ld_bytes;
    float bv = -INFINITY;
    int bi = kIdxSentinel;
    for (int c = c0; c < c0 + nch; ++c) {
      const int cbase = c * CE;
      float x[EPT];
#pragma unroll
      for (int j = 0; j < kVecPerThread; ++j) {
        int e0 = cbase + (j * kStreamThreads + tid) * EPV;
        uint4 v;
        if (ALIGNED && e0 + EPV <= V) {
          v = ldg_stream(rp + (size_t)e0 * ESZ);
          uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            if (BF16) {
              x[j * 8 + 2 * q2] = __uint_as_float(w[q2] << 16);
              x[j * 8 + 2 * q2 + 1] = __uint_as_float(w[q2] & 0xffff0000u);
            } else {
              x[j * 4 + q2] = __uint_as_float(w[q2]);
            }
          }
        } else {
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
        int gi = cbase + ((n / EPV) * kStreamThreads + tid) * EPV + (n % EPV);
        if (x[n] == m && mi == kIdxSentinel && gi < V) mi = gi;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(kFull, m, o);
        int oi = __shfl_xor_sync(kFull, mi, o);
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
    __syncthreads();
    if (tid == 0) {
      float v = sh.wv[0];
      int ix = sh.wi[0];
      for (int w = 1; w < kStreamWarps; ++w)
        if (better(sh.wv[w], sh.wi[w], v, ix)) {
          v = sh.wv[w];
          ix = sh.wi[w];
        }
      size_t so = (size_t)row * cpr + c0;
      P.vsegv[so] = v;
      P.vsegi[so] = ix;
      P.vseglen[so] = nch;
      __threadfence();
      int old = atomicAdd(&P.row_done[row], nch);
      sh.last = (old + nch == cpr);
    }
    __syncthreads();
    if (sh.last) {
      // merge this row's segments (warp 0)
      if (warp == 0) {
        __threadfence();
        float v = -INFINITY;
        int ix = kIdxSentinel;
        for (int c = lane; c < cpr; c += 32) {
          size_t so = (size_t)row * cpr + c;
          if (__ldcg(&P.vseglen[so]) > 0) {
            float sv = __ldcg(&P.vsegv[so]);
            int si = __ldcg(&P.vsegi[so]);
            if (better(sv, si, v, ix)) {
              v = sv;
              ix = si;
            }
            P.vseglen[so] = 0;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          float ov = __shfl_xor_sync(kFull, v, o);
          int oi = __shfl_xor_sync(kFull, ix, o);
          if (better(ov, oi, v, ix)) {
            v = ov;
            ix = oi;
          }
        }
        if (lane == 0) {
          P.vrow_arg[(size_t)r * T + i] = ix;
          P.row_done[row] = 0;
          __threadfence();
          int old = atomicAdd(&P.req_done[r], 1);
          sh.rlast = (old + 1 == P.n_nodes[r]);
        }
        __syncwarp();
        if (sh.rlast) {
          // greedy walk of request r
          __threadfence();
          const int n = P.n_nodes[r];
          const int D = P.d > 0 ? P.d : 1;
          int cur = 0, acc = 0, bon = -1;
          for (;;) {
            int t = __ldcg(&P.vrow_arg[(size_t)r * T + cur]);
            int found = -1;
            for (int j0 = cur + 1; j0 < n; j0 += 32) {
              int j = j0 + lane;
              bool f = j < n && P.parent[(size_t)r * T + j] == cur && P.tok[(size_t)r * T + j] == t;
              unsigned bal = __ballot_sync(kFull, f);
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
      __syncthreads();
    }
    q += nch;
  }
  if (nanf) atomicOr(P.err, kErrTargetNaN);
}

}  // namespace

void launch_mask(const Params& P, uint32_t* mask, int32_t* pos, int32_t* parent, int32_t* tok, int32_t* tree_len,
                 cudaStream_t s) {
  mask_kernel<<<1, 1024, 0, s>>>(P, mask, pos, parent, tok, tree_len);
}

int verify_occupancy() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, verify_kernel<true, true>, kStreamThreads, 0);
  return n > 0 ? n : 1;
}

void launch_verify(const Params& P, const void* target, long long ld_bytes, bool aligned, int32_t* accept_len,
                   int32_t* accept_path, int32_t* bonus, int grid, cudaStream_t s) {
  const char* t = static_cast<const char*>(target);
  if (P.dtype == SMART_BF16) {
    if (aligned) verify_kernel<true, true><<<grid, kStreamThreads, 0, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
    else verify_kernel<true, false><<<grid, kStreamThreads, 0, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
  } else {
    if (aligned) verify_kernel<false, true><<<grid, kStreamThreads, 0, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
    else verify_kernel<false, false><<<grid, kStreamThreads, 0, s>>>(P, t, ld_bytes, accept_len, accept_path, bonus);
  }
}

}  // namespace smart
