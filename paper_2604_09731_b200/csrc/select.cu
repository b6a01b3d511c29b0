// select.cu — K2 `smart_select`: A3 marginal benefit + per-request eligibility, A4 batch-global
// ranking, A5 prefix scan + decision rule, A6 commit of A_l and the next frontier.
//
// PAPER.md: marginal benefit Eq.(13), marginal cost Eq.(15), rule
// Eq.(12)/(16) P:294-300/Algorithm 1 lines 5-12 P:859-871, budget Eq.(8) P:243.
// Readings: Q3 (mid-layer budget cut), Q6 (|P| frozen at layer start), Q7 (FROZEN/PREFIX),
// Q8 (strict >), Q9 (ties), Q13 (batch-coupled cost), Q19 (omega).
//
// One CTA of 1024 threads: the work is latency-bound (<= 16 K candidates).  Keys are 64-bit
// (~orderable(b) | global request | c) so an ascending bitonic sort gives (b desc, r asc, c asc)
// and every record is self-describing (no payload) — the same keys are what ranks exchange
// over NCCL when the batch is sharded (phase 0 -> all-gather -> phase 1).
// All selection arithmetic is fp64; E0 is summed in global request order (partition-invariant).
#include "smart_internal.cuh"

namespace smart {

namespace {

__device__ __forceinline__ unsigned long long sel_key(float b, int r_glob, int c) {
  return ((unsigned long long)(~float_orderable(b)) << 32) | ((unsigned long long)(unsigned)r_glob << 16) |
         (unsigned long long)(unsigned)c;
}
__device__ __forceinline__ float key_b(unsigned long long key) {
  uint32_t o = ~(uint32_t)(key >> 32);
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}
__device__ __forceinline__ int key_r(unsigned long long key) { return (int)((key >> 16) & 0xffffu); }
__device__ __forceinline__ int key_c(unsigned long long key) { return (int)(key & 0xffffu); }

struct SelShared {
  double dred[32];
  int ired[32];
  double dtmp[8];
  int itmp[8];
  int ne, jstar, argj;
};

// block-wide exclusive scan of ints in smem arr[0..n) (n <= 1024 * items); returns total
__device__ int block_excl_scan_int(int* arr, int n, SelShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + kSelectThreads - 1) / kSelectThreads;
  const int b0 = tid * per, b1 = min(n, b0 + per);
  int local = 0;
  for (int i = b0; i < b1; ++i) local += arr[i];
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sh.ired[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = sh.ired[lane];
    int iv = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(kFull, iv, o);
      if (lane >= o) iv += t;
    }
    sh.ired[lane] = iv - v;  // exclusive warp offsets
    if (lane == 31) sh.itmp[0] = iv;
  }
  __syncthreads();
  int run = sh.ired[warp] + incl - local;
  for (int i = b0; i < b1; ++i) {
    int v = arr[i];
    arr[i] = run;
    run += v;
  }
  int total = sh.itmp[0];
  __syncthreads();
  return total;
}

// ascending bitonic sort of keys[0..P2), P2 a power of two
__device__ void block_bitonic(unsigned long long* keys, int P2) {
  const int tid = threadIdx.x;
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < (P2 >> 1); i += kSelectThreads) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool asc = (lo & size) == 0;
        unsigned long long a = keys[lo], b = keys[hi];
        if ((a > b) == asc) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// A3 for the local requests: writes each request's eligible candidates (sorted within the
// request) into keys[base_r + rank]; returns the local eligible count.  Also stores b.
__device__ int local_eligible(const Params& P, int layer, unsigned long long* keys, int* s_e, SelShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1;
  const int k = P.k;
  const size_t lbase = (size_t)(layer - 1) * P.cap_rows * k;
  for (int r = tid; r < P.b_loc; r += kSelectThreads) {
    int nc = P.fr_cnt[par][r] * k;
    int q = P.B - (P.n_nodes[r] - 1);
    if (q > P.Wq) q = P.Wq;
    if (q < 0) q = 0;
    s_e[r] = min(q, nc);
  }
  __syncthreads();
  int ne = block_excl_scan_int(s_e, P.b_loc, sh);
  // per request (one warp each): benefit, within-request rank by (b desc, c asc)
  for (int r = warp; r < P.b_loc; r += kSelectThreads / 32) {
    const int nc = P.fr_cnt[par][r] * k;
    if (nc == 0) continue;
    const size_t cb = lbase + (size_t)P.fr_off[par][r] * k;
    const float D = (P.accept_model == SMART_PATH_MEAN) ? (float)P.leaf_cnt[r] : 1.f;  // Eq.(13), Q6
    const int e_r = (r + 1 < P.b_loc ? s_e[r + 1] : ne) - s_e[r];
    for (int i0 = 0; i0 < nc; i0 += 32) {
      int i = i0 + lane;
      float bi = -1.f;
      if (i < nc) {
        bi = __fdiv_rn(P.cand[cb + i].cum, D);
        P.cand_b[cb + i] = bi;
        P.cand_adm[cb + i] = 0;
      }
      int rank = 0;
      for (int j0 = 0; j0 < nc; j0 += 32) {
        int j = j0 + lane;
        float bj_reg = (j < nc) ? __fdiv_rn(P.cand[cb + j].cum, D) : -2.f;
        int lim = min(32, nc - j0);
        for (int t = 0; t < lim; ++t) {
          float bj = __shfl_sync(kFull, bj_reg, t);
          int jj = j0 + t;
          rank += (bj > bi) || (bj == bi && jj < i);
        }
      }
      if (i < nc && rank < e_r) keys[s_e[r] + rank] = sel_key(bi, P.b_off + r, i);
    }
  }
  __syncthreads();
  return ne;
}

// A5 over sorted keys[0..ne): decision rule and first failure j*, argmax_j S_j.
__device__ void scan_and_cut(const Params& P, const unsigned long long* keys, int ne, long long N0, double E0,
                             int b_cost, DevTrace& tr, SelShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int sat = 0;
  const double Sb0 = speed_b(P, E0, N0, b_cost, &sat);
  const double dc0 = marginal_cost(P, N0, &sat);
  const double ac = P.alpha * P.c_T;
  const int per = (ne + kSelectThreads - 1) / kSelectThreads;
  const int j0 = tid * per, j1 = min(ne, j0 + per);
  // exclusive prefix sums of b in sorted order (fp64)
  double local = 0.0;
  for (int j = j0; j < j1; ++j) local += (double)key_b(keys[j]);
  double incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sh.dred[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double v = sh.dred[lane];
    double iv = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t = __shfl_up_sync(kFull, iv, o);
      if (lane >= o) iv += t;
    }
    sh.dred[lane] = iv - v;
  }
  __syncthreads();
  double run = sh.dred[warp] + incl - local;  // sum of b over positions < j0
  int first_fail = ne;
  double bestS = -1.0;
  int bestj = ne + 1;
  for (int j = j0; j < j1; ++j) {
    double bj = (double)key_b(keys[j]);
    bool ok;
    if (P.selection == SMART_FROZEN) {
      ok = ac * bj / dc0 > Sb0;                                  // Alg.1 frozen globals
    } else {
      long long Nj = N0 + j;
      double Sj = speed_b(P, E0 + run, Nj, b_cost, &sat);        // S_{j-1}
      double dcj = marginal_cost(P, Nj, &sat);
      ok = ac * bj / dcj > Sj;                                   // Eq.(16), strict
    }
    if (!ok && j < first_fail) first_fail = j;
    run += bj;
    double Safter = speed_b(P, E0 + run, N0 + j + 1, b_cost, &sat);
    if (Safter > bestS) {
      bestS = Safter;
      bestj = j + 1;
    }
  }
  // block min of first_fail; block argmax (value desc, index asc) of S_j
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    first_fail = min(first_fail, __shfl_xor_sync(kFull, first_fail, o));
    double os = __shfl_xor_sync(kFull, bestS, o);
    int oj = __shfl_xor_sync(kFull, bestj, o);
    if (os > bestS || (os == bestS && oj < bestj)) {
      bestS = os;
      bestj = oj;
    }
  }
  __syncthreads();
  if (lane == 0) {
    sh.ired[warp] = first_fail;
    sh.dred[warp] = bestS;
  }
  __shared__ int s_bj[32];
  if (lane == 0) s_bj[warp] = bestj;
  const int any_sat = __syncthreads_or(sat);
  if (any_sat && tid == 0) atomicOr(P.err, kErrSaturated);
  if (tid == 0) {
    int ff = ne;
    double bs = Sb0;
    int bj = 0;  // j = 0: the empty prefix
    for (int w = 0; w < 32; ++w) {
      ff = min(ff, sh.ired[w]);
      if (sh.dred[w] > bs || (sh.dred[w] == bs && s_bj[w] < bj)) {
        bs = sh.dred[w];
        bj = s_bj[w];
      }
    }
    sh.jstar = ff;
    sh.argj = bj;
    tr.N0 = (int)N0;
    tr.E0 = E0;
    tr.S0 = Sb0 / b_cost;
    tr.dc0 = dc0;
    tr.n_admit = ff;
    tr.argmax_j = bj;
    tr.saturated = any_sat ? 1 : 0;
  }
  __syncthreads();
}

// A6: commit admitted candidates of the local requests; next frontier; E_r bookkeeping.
__device__ void commit(const Params& P, int layer, int* s_cnt, SelShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1, npar = layer & 1;
  const int k = P.k;
  const size_t lbase = (size_t)(layer - 1) * P.cap_rows * k;
  // pass 1: admitted count per request
  for (int r = warp; r < P.b_loc; r += kSelectThreads / 32) {
    const int nc = P.fr_cnt[par][r] * k;
    const size_t cb = lbase + (size_t)P.fr_off[par][r] * k;
    int a = 0;
    for (int i = lane; i < nc; i += 32) a += P.cand_adm[cb + i];
    a = warp_sum_i(a);
    if (lane == 0) {
      int nd = P.n_nodes[r] - 1 + a;
      bool fin = P.finished[r] || a == 0 || nd >= P.B;  // Alg.1 line 10
      s_cnt[r] = fin ? 0 : a;
      s_cnt[P.b_loc + r] = a;
    }
  }
  __syncthreads();
  // next frontier offsets (exclusive scan of next counts)
  for (int r = tid; r < P.b_loc; r += kSelectThreads) P.fr_cnt[npar][r] = s_cnt[r];
  __syncthreads();
  int total = block_excl_scan_int(s_cnt, P.b_loc, sh);
  for (int r = tid; r < P.b_loc; r += kSelectThreads) P.fr_off[npar][r] = s_cnt[r];
  if (tid == 0) *P.fr_total[npar] = total;
  // pass 2: write nodes in canonical order (c asc), frontier entries, E_r
  for (int r = warp; r < P.b_loc; r += kSelectThreads / 32) {
    const int nc = P.fr_cnt[par][r] * k;
    const size_t cb = lbase + (size_t)P.fr_off[par][r] * k;
    const int a_tot = s_cnt[P.b_loc + r];
    if (a_tot == 0) {
      if (lane == 0 && nc > 0) P.finished[r] = 1;
      continue;
    }
    const int n0 = P.n_nodes[r];
    const bool to_frontier = P.fr_cnt[npar][r] > 0;
    const int foff = P.fr_off[npar][r];
    int a = 0;
    double esum = 0.0, psum_new = 0.0, psum_par = 0.0;
    int npar_exp = 0;
    for (int i0 = 0; i0 < nc; i0 += 32) {
      int i = i0 + lane;
      bool f = (i < nc) && P.cand_adm[cb + i];
      unsigned bal = __ballot_sync(kFull, f);
      int pre = __popc(bal & ((1u << lane) - 1u));
      if (f) {
        Cand cd = P.cand[cb + i];
        int node = n0 + a + pre;
        size_t o = (size_t)r * P.T + node;
        P.tok[o] = cd.tok;
        P.parent[o] = cd.parent;
        P.depth[o] = layer;
        P.p[o] = cd.p;
        P.cum[o] = cd.cum;
        esum += (double)cd.cum;
        if (P.accept_model == SMART_PATH_MEAN) {
          double ps = P.path_sum[(size_t)r * P.T + cd.parent] + (double)cd.cum;
          P.path_sum[o] = ps;
          psum_new += ps;
        }
        if (to_frontier) P.fr[npar][foff + a + pre] = make_int2(r, node);
      }
      // distinct parents that received children: first admitted candidate of each row group
      if (P.accept_model == SMART_PATH_MEAN && f) {
        int rank_in_row = i % k;
        bool first = true;
        for (int j = i - rank_in_row; j < i; ++j)
          if (P.cand_adm[cb + j]) { first = false; break; }
        if (first) {
          psum_par += P.path_sum[(size_t)r * P.T + P.cand[cb + i].parent];
          npar_exp += 1;
        }
      }
      a += __popc(bal);
    }
    esum = warp_sum_d(esum);
    psum_new = warp_sum_d(psum_new);
    psum_par = warp_sum_d(psum_par);
    npar_exp = warp_sum_i(npar_exp);
    if (lane == 0) {
      P.n_nodes[r] = n0 + a;
      if (P.accept_model == SMART_PATH_MEAN) {
        int lc = P.leaf_cnt[r] - npar_exp + a;
        double ls = P.leaf_sum[r] - psum_par + psum_new;
        P.leaf_cnt[r] = lc;
        P.leaf_sum[r] = ls;
        P.E_r[r] = ls / (double)lc;  // Eq.(2) path mean
      } else {
        P.E_r[r] += esum;            // node sum (Q11)
      }
      if (!to_frontier) P.finished[r] = 1;
    }
  }
  __syncthreads();
}

// sums over local requests in request order (single thread; fp64)
__device__ void local_totals(const Params& P, long long& N, double& E) {
  N = 0;
  E = 0.0;
  for (int r = 0; r < P.b_loc; ++r) {
    N += P.n_nodes[r] - 1;
    E += P.E_r[r];
  }
}

// phase 2: single rank (or LOCAL cost scope).  phase 0: local part + pack exchange buffers.
// phase 1: merge gathered buffers, cut, commit own.
__global__ void __launch_bounds__(kSelectThreads, 1) select_kernel(Params P, int layer, int phase) {
  extern __shared__ unsigned long long smem_keys[];
  __shared__ SelShared sh;
  const int tid = threadIdx.x;
  const int par = (layer - 1) & 1;
  const int R = *P.fr_total[par];
  DevTrace& tr = P.trace[layer - 1];
  int* s_int = reinterpret_cast<int*>(smem_keys);  // reused region for per-request ints

  if (phase == 2 && R == 0) {
    // no frontier anywhere: the step has terminated (A_{l-1} empty)
    if (tid == 0) {
      tr.executed = 0;
      *P.fr_total[layer & 1] = 0;
    }
    for (int r = tid; r < P.b_loc; r += kSelectThreads) P.fr_cnt[layer & 1][r] = 0;
    return;
  }
  // keys region after 2*b_loc ints (aligned to 8 bytes)
  unsigned long long* keys = smem_keys + (2 * P.b_loc + 1) / 2 + 1;

  if (phase == 0 || phase == 2) {
    int ne = local_eligible(P, layer, keys, s_int, sh);
    if (phase == 2) {
      int P2 = 1;
      while (P2 < ne) P2 <<= 1;
      for (int i = ne + tid; i < P2; i += kSelectThreads) keys[i] = ~0ull;
      __syncthreads();
      block_bitonic(keys, P2);
      long long N0;
      double E0;
      __shared__ long long sN;
      __shared__ double sE;
      if (tid == 0) {
        local_totals(P, N0, E0);
        sN = N0;
        sE = E0;
        tr.executed = 1;
        tr.n_rows = R;
        tr.n_cand = R * P.k;
        tr.n_elig = ne;
      }
      __syncthreads();
      N0 = sN;
      E0 = sE;
      scan_and_cut(P, keys, ne, N0, E0, P.cost_scope == SMART_COST_LOCAL ? P.b_loc : P.b_glob, tr, sh);
      const int js = sh.jstar;
      const size_t lbase = (size_t)(layer - 1) * P.cap_rows * P.k;
      for (int j = tid; j < js; j += kSelectThreads) {
        unsigned long long key = keys[j];
        int r = key_r(key) - P.b_off;
        P.cand_adm[lbase + (size_t)P.fr_off[par][r] * P.k + key_c(key)] = 1;
      }
      __syncthreads();
      commit(P, layer, s_int, sh);
      if (tid == 0) {
        long long N;
        double E;
        local_totals(P, N, E);
        int s2 = 0;
        int bc = P.cost_scope == SMART_COST_LOCAL ? P.b_loc : P.b_glob;
        tr.S_after = speed_b(P, E, N, bc, &s2) / bc;
        *P.N_glob = (int)N;
        *P.E_glob = E;
      }
      return;
    }
    // phase 0: sort local eligible, pack exchange buffers (keys padded with ~0)
    int P2 = 1;
    while (P2 < ne) P2 <<= 1;
    for (int i = ne + tid; i < P2; i += kSelectThreads) keys[i] = ~0ull;
    __syncthreads();
    block_bitonic(keys, P2);
    unsigned long long* xk = reinterpret_cast<unsigned long long*>(P.xs);
    double* xE = reinterpret_cast<double*>(P.xs + (size_t)P.m_cap * 8);
    int* xh = reinterpret_cast<int*>(P.xs + (size_t)P.m_cap * 8 + (size_t)P.b_loc * 8);
    for (int i = tid; i < P.m_cap; i += kSelectThreads) xk[i] = i < ne ? keys[i] : ~0ull;
    for (int r = tid; r < P.b_loc; r += kSelectThreads) {
      xh[r] = P.n_nodes[r] - 1;
      xE[r] = P.E_r[r];
    }
    if (tid == 0) xh[P.b_loc] = ne;
    return;
  }

  // ---- phase 1: global merge over all ranks ----
  const int tot = P.nranks * P.m_cap;
  int P2 = 1;
  while (P2 < tot) P2 <<= 1;
  for (int i = tid; i < P2; i += kSelectThreads) {
    unsigned long long v = ~0ull;
    if (i < tot) {
      int g = i / P.m_cap, e = i % P.m_cap;
      v = reinterpret_cast<const unsigned long long*>(P.xr + (size_t)g * P.xstride)[e];
    }
    keys[i] = v;
  }
  __syncthreads();
  block_bitonic(keys, P2);
  __shared__ long long gN;
  __shared__ double gE;
  __shared__ int gne, grows;
  if (tid == 0) {
    long long N = 0;
    double E = 0.0;
    int ne = 0;
    for (int g = 0; g < P.nranks; ++g) {
      const char* rec = P.xr + (size_t)g * P.xstride;
      const double* xE = reinterpret_cast<const double*>(rec + (size_t)P.m_cap * 8);
      const int* h = reinterpret_cast<const int*>(rec + (size_t)P.m_cap * 8 + (size_t)P.b_loc * 8);
      for (int r = 0; r < P.b_loc; ++r) {
        N += h[r];
        E += xE[r];  // global request order (ranks own contiguous request ranges)
      }
      ne += h[P.b_loc];
    }
    gN = N;
    gE = E;
    gne = ne;
    grows = R;
    tr.executed = 1;
    tr.n_rows = R;
    tr.n_cand = R * P.k;
    tr.n_elig = ne;
  }
  __syncthreads();
  const int ne = gne;
  if (ne == 0 && R == 0) {
    // nothing anywhere at this layer
  }
  scan_and_cut(P, keys, ne, gN, gE, P.b_glob, tr, sh);
  const int js = sh.jstar;
  const size_t lbase = (size_t)(layer - 1) * P.cap_rows * P.k;
  // clear local admitted flags, then mark own admitted
  for (int i = tid; i < R * P.k; i += kSelectThreads) P.cand_adm[lbase + i] = 0;
  __syncthreads();
  for (int j = tid; j < js; j += kSelectThreads) {
    unsigned long long key = keys[j];
    int r = key_r(key) - P.b_off;
    if (r >= 0 && r < P.b_loc) P.cand_adm[lbase + (size_t)P.fr_off[par][r] * P.k + key_c(key)] = 1;
  }
  __syncthreads();
  commit(P, layer, s_int, sh);
  __syncthreads();
  if (tid == 0) {
    // S_after needs the global E, N after the layer: recompute from the pre-layer globals and
    // the admitted prefix (identical on every rank).
    double Ea = gE;
    for (int j = 0; j < js; ++j) Ea += (double)key_b(keys[j]);
    long long Na = gN + js;
    int s2 = 0;
    if (P.accept_model == SMART_NODE_SUM) tr.S_after = speed_b(P, Ea, Na, P.b_glob, &s2) / P.b_glob;
    *P.N_glob = (int)Na;
    *P.E_glob = Ea;
  }
}

__global__ void export_frontier_kernel(Params P, int parity, int32_t* out, int32_t* count) {
  int n = *P.fr_total[parity];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; out && i < n; i += gridDim.x * blockDim.x) {
    int2 e = P.fr[parity][i];
    out[2 * i] = e.x;
    out[2 * i + 1] = e.y;
  }
  if (count && blockIdx.x == 0 && threadIdx.x == 0) *count = n;
}

}  // namespace

size_t select_smem_bytes(int sort_cap) {
  // per-request ints (2*b_loc) are accounted by the caller via sort_cap padding
  return (size_t)sort_cap * 8;
}

void launch_select(const Params& P, int layer, int phase, size_t smem, cudaStream_t s) {
  select_kernel<<<1, kSelectThreads, smem, s>>>(P, layer, phase);
}

void launch_export_frontier(const Params& P, int parity, int32_t* d_frontier, int32_t* d_count, cudaStream_t s) {
  if (d_frontier) export_frontier_kernel<<<8, 256, 0, s>>>(P, parity, d_frontier, d_count);
  else if (d_count) export_frontier_kernel<<<1, 32, 0, s>>>(P, parity, nullptr, d_count);
}

cudaError_t select_set_smem(size_t bytes) {
  return cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace smart
