// select_core.cuh — A3-A6 of one layer as a block-level device routine (any block size that is a
// multiple of 32).  Called (a) by the last CTA of the fused layer kernel (256 consumer threads)
// and (b) by the standalone select kernel (multi-rank phases, very large batches).
//
// PAPER.md: marginal benefit Eq.(13); marginal cost Eq.(15); decision rule
// Eq.(12)/(16) P:294-300 / P:347-355; Algorithm 1 lines 5-12 P:859-871; budget Eq.(8) P:243.
// Readings: Q3 mid-layer budget cut, Q6 |P| frozen at layer start, Q7 FROZEN/PREFIX, Q8 strict >,
// Q9 ties (b desc, request asc, c asc), Q13 batch-coupled cost, Q19 omega.
//
// Determinism: every floating-point reduction has a structure fixed by the data size only
// (32-wide xor/up trees per tile, sequential over tiles), never by the block size or by how the
// batch is sharded — G ranks reproduce the G = 1 decisions bit for bit.
#pragma once

#include "smart_internal.cuh"

namespace smart {

// barrier among the NT threads running the selection: named barrier 1 (the fused layer kernel's
// producer warp never joins it; in the standalone kernel NT == blockDim.x)
template <int NT>
__device__ __forceinline__ void blk_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

enum SelectMode { kSelFull = 0, kSelLocal = 1, kSelGlobal = 2 };
constexpr int kA5Par = 256;  // A5 lists up to this length: one entry per thread (<= every NT used)

__device__ __forceinline__ unsigned long long sel_key(float b, int r_glob, int c) {
  return ((unsigned long long)(~float_orderable(b)) << 32) | ((unsigned long long)(unsigned)r_glob << 16) |
         (unsigned long long)(unsigned)c;
}
__device__ __forceinline__ float sel_key_b(unsigned long long key) {
  uint32_t o = ~(uint32_t)(key >> 32);
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}
__device__ __forceinline__ int sel_key_r(unsigned long long key) { return (int)((key >> 16) & 0xffffu); }
__device__ __forceinline__ int sel_key_c(unsigned long long key) { return (int)(key & 0xffffu); }

// b * S = c_T (omega b + E) / cost(N), cost from the host-built fp64 table (0/0 := 0, Q4)
__device__ __forceinline__ double speed_tab(const Params& P, double E, long long N, int b) {
  double C = P.cost_tab[N];
  return C > 0.0 ? P.c_T * ((double)P.omega * b + E) / C : 0.0;
}

struct SelScratch {
  double tile_d[260];
  int tile_i[1040];
  double bcast_d[4];
  long long bcast_l[2];
  int bcast_i[8];
  int wred_i[32];
  double wred_d[32];
};

// ---- deterministic, block-size independent helpers -----------------------------------------

// sum of a[0..n) (smem): 32-wide xor trees per tile, tiles summed in order by one thread
template <int NT>
__device__ double det_sum(const double* a, int n, SelScratch& ss) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntile = (n + 31) / 32;
  for (int t = warp; t < ntile; t += NT / 32) {
    int i = t * 32 + lane;
    double v = i < n ? a[i] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) ss.tile_d[t] = v;
  }
  blk_sync<NT>();
  if (tid == 0) {
    double s = 0.0;
    for (int t = 0; t < ntile; ++t) s += ss.tile_d[t];
    ss.bcast_d[0] = s;
  }
  blk_sync<NT>();
  double r = ss.bcast_d[0];
  blk_sync<NT>();
  return r;
}

template <int NT>
__device__ long long block_sum_ll(long long v, SelScratch& ss) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  blk_sync<NT>();
  if (lane == 0) ss.wred_d[warp] = (double)v;  // exact for counts < 2^53
  blk_sync<NT>();
  if (tid == 0) {
    double s = 0;
    for (int w = 0; w < NT / 32; ++w) s += ss.wred_d[w];
    ss.bcast_l[0] = (long long)s;
  }
  blk_sync<NT>();
  long long r = ss.bcast_l[0];
  blk_sync<NT>();
  return r;
}

// exclusive scan of ints in smem a[0..n) in place; returns total (ints: association-free)
template <int NT>
__device__ int excl_scan_int(int* a, int n, SelScratch& ss) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntile = (n + 31) / 32;
  for (int t = warp; t < ntile; t += NT / 32) {
    const int i = t * 32 + lane;
    const int v = i < n ? a[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += u;
    }
    if (i < n) a[i] = incl - v;
    if (lane == 31) ss.tile_i[t] = incl;
  }
  blk_sync<NT>();
  if (warp == 0) {
    // tile totals: each lane owns a contiguous group of tiles, then one warp scan
    const int per = (ntile + 31) / 32;
    const int t0 = lane * per, t1 = min(ntile, t0 + per);
    int loc = 0;
    for (int t = t0; t < t1; ++t) loc += ss.tile_i[t];
    int incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += u;
    }
    int run = incl - loc;
    for (int t = t0; t < t1; ++t) {
      const int v = ss.tile_i[t];
      ss.tile_i[t] = run;
      run += v;
    }
    if (lane == 31) ss.bcast_i[0] = incl;
  }
  blk_sync<NT>();
  for (int i = tid; i < n; i += NT) a[i] += ss.tile_i[i >> 5];
  const int total = ss.bcast_i[0];
  blk_sync<NT>();
  return total;
}

// ascending bitonic sort of keys[0..P2) (P2 power of two)
template <int NT>
__device__ void bitonic_sort(unsigned long long* keys, int P2) {
  const int tid = threadIdx.x;
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < (P2 >> 1); i += NT) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool asc = (lo & size) == 0;
        unsigned long long a = keys[lo], b = keys[hi];
        if ((a > b) == asc) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
      blk_sync<NT>();
    }
  }
}

// ascending bitonic sort of keys[0..P2) with two keys per thread (P2 <= 2*NT, power of two):
// strides < 32 exchange by shuffles, stride 32 inside the thread, strides >= 64 through shared
// memory (2 barriers each).  Element i lives in warp i/64, register (i%64)/32, lane i%32.
template <int NT>
__device__ void bitonic_sort_reg(unsigned long long* keys, int P2) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = warp * 64 + lane, i1 = i0 + 32;
  const bool act = i0 < P2;
  unsigned long long v0 = act ? keys[i0] : ~0ull, v1 = act ? keys[i1] : ~0ull;
  auto cx_reg = [](unsigned long long& a, unsigned long long& b, bool asc) {  // a at lower index
    const bool sw = (a > b) == asc;
    const unsigned long long t = sw ? b : a;
    b = sw ? a : b;
    a = t;
  };
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 64) {
        blk_sync<NT>();  // previous readers done
        if (act) {
          keys[i0] = v0;
          keys[i1] = v1;
        }
        blk_sync<NT>();
        if (act) {
          const int p0 = i0 ^ stride, p1 = i1 ^ stride;
          const unsigned long long o0 = keys[p0], o1 = keys[p1];
          const bool asc0 = (i0 & size) == 0, asc1 = (i1 & size) == 0;
          // keep min if (lower index) == asc, else max
          v0 = ((i0 < p0) == asc0) ? (v0 < o0 ? v0 : o0) : (v0 > o0 ? v0 : o0);
          v1 = ((i1 < p1) == asc1) ? (v1 < o1 ? v1 : o1) : (v1 > o1 ? v1 : o1);
        }
      } else if (stride == 32) {
        const bool asc = (i0 & size) == 0;  // i0 and i1 = i0 + 32 share the direction bit (size >= 64)
        cx_reg(v0, v1, asc);
      } else {
        const unsigned long long o0 = __shfl_xor_sync(kFull, v0, stride);
        const unsigned long long o1 = __shfl_xor_sync(kFull, v1, stride);
        const bool lo = (lane & stride) == 0;
        const bool asc0 = (i0 & size) == 0, asc1 = (i1 & size) == 0;
        v0 = (lo == asc0) ? (v0 < o0 ? v0 : o0) : (v0 > o0 ? v0 : o0);
        v1 = (lo == asc1) ? (v1 < o1 ? v1 : o1) : (v1 > o1 ? v1 : o1);
      }
    }
  }
  blk_sync<NT>();
  if (act) {
    keys[i0] = v0;
    keys[i1] = v1;
  }
  blk_sync<NT>();
}

// ---- layout of the dynamic shared memory used by select_layer --------------------------------
// Per candidate only its benefit (4 B) is staged; records are re-read from global (L2) at commit.
// Admitted candidates are per-request bitmaps (bit c = candidate index within the request).
struct SelLayout {
  int* cnt;       // [b_loc] frontier rows of the layer per request
  int* off;       // [b_loc] frontier offset
  int* nd;        // [b_loc] drafted nodes before the layer
  int* base;      // [b_loc] eligible base (A3), later next-frontier offsets
  int* adm;       // [b_loc] admitted per request
  int* nxt;       // [b_loc] next-frontier count per request
  int* fin;       // [b_loc] finished flag
  float* D;       // [b_loc] benefit divisor |P_r| (PATH_MEAN) or 1
  unsigned* bm;   // [b_loc * nbw] admitted bitmaps
  int* rreq;      // [cap_rows] request of each frontier row
  float* cb;      // [nc_cap] benefit of each candidate
  float* cslot;   // [b_loc * wf] cum of the request's admits (index order)
  double* pslot;  // [b_loc * wf] parent path sum of the request's admits (PATH_MEAN)
  double* ctab;   // [sort_cap + 2] cost(N0 + j)
  double* dtab;   // [sort_cap + 2] marginal cost at N0 + j
  double* E;      // [b_all] E_r (global order in kSelGlobal)
  unsigned long long* keys;   // [sort_cap]
  unsigned long long* keys2;  // [sort_cap] rank-sort output / scratch
  int nbw, wf;
};

__host__ __device__ inline size_t sel_align(size_t x) { return (x + 15) & ~size_t(15); }

// nc_cap = cap_rows * k = b_loc * wf * k
// staged candidate records (P.sel_rec): 16 B per candidate, after keys2
__host__ __device__ inline size_t sel_rec_bytes(int nc_cap) { return (size_t)nc_cap * 16; }

// bucket sort scratch for lists longer than 256 keys (2 x kSortBuckets ints, after the records)
constexpr int kSortBucketBits = 12;
constexpr int kSortBuckets = 1 << kSortBucketBits;
__host__ __device__ inline size_t sel_bucket_bytes(int sort_cap) {
  return sort_cap > 256 ? (size_t)2 * kSortBuckets * 4 : 0;
}

__host__ __device__ inline size_t sel_smem_bytes(int b_loc, int b_all, int sort_cap, int nc_cap, int nranks = 1,
                                                 int k = 1) {
  const int per_req = nc_cap / (b_loc > 0 ? b_loc : 1);  // wf * k
  const int nbw = (per_req + 31) / 32;
  const int wf = per_req / (k > 0 ? k : 1);
  size_t bytes = sel_align((size_t)8 * b_loc * 4);
  bytes += sel_align((size_t)b_loc * nbw * 4);
  bytes += sel_align((size_t)(nc_cap / (k > 0 ? k : 1)) * 4);
  bytes += sel_align((size_t)nc_cap * 4);
  bytes += sel_align((size_t)b_loc * wf * 4);
  bytes += sel_align((size_t)b_loc * wf * 8);
  bytes += sel_align(((size_t)sort_cap + 2) * 16);
  bytes += sel_align((size_t)b_all * 8);
  bytes += (size_t)sort_cap * 16;
  bytes += sel_bucket_bytes(sort_cap);  // (after the staged records, when those are present)
  (void)nranks;
  return bytes;
}

__device__ inline SelLayout sel_layout(char* smem, int b_loc, int nc_cap, int k, int sort_cap) {
  SelLayout L;
  const int per_req = nc_cap / b_loc;
  L.nbw = (per_req + 31) / 32;
  L.wf = per_req / k;
  int* ip = reinterpret_cast<int*>(smem);
  L.cnt = ip;
  L.off = ip + b_loc;
  L.nd = ip + 2 * b_loc;
  L.base = ip + 3 * b_loc;
  L.adm = ip + 4 * b_loc;
  L.nxt = ip + 5 * b_loc;
  L.fin = ip + 6 * b_loc;
  L.D = reinterpret_cast<float*>(ip + 7 * b_loc);
  size_t o = sel_align((size_t)8 * b_loc * 4);
  L.bm = reinterpret_cast<unsigned*>(smem + o);
  o += sel_align((size_t)b_loc * L.nbw * 4);
  L.rreq = reinterpret_cast<int*>(smem + o);
  o += sel_align((size_t)(nc_cap / k) * 4);
  L.cb = reinterpret_cast<float*>(smem + o);
  o += sel_align((size_t)nc_cap * 4);
  L.cslot = reinterpret_cast<float*>(smem + o);
  o += sel_align((size_t)b_loc * L.wf * 4);
  L.pslot = reinterpret_cast<double*>(smem + o);
  o += sel_align((size_t)b_loc * L.wf * 8);
  L.ctab = reinterpret_cast<double*>(smem + o);
  L.dtab = L.ctab + sort_cap + 2;
  o += sel_align(((size_t)sort_cap + 2) * 16);
  L.E = reinterpret_cast<double*>(smem + o);
  return L;
}

// warp-level exclusive scan of per-request ints held lane-blocked: lane l owns requests
// [l*per, min(n, (l+1)*per)) stored in smem a[]; returns the total (ints: association-free)
__device__ __forceinline__ int warp_excl_scan_smem(int* a, int n, int lane) {
  const int per = (n + 31) / 32;
  const int r0 = lane * per, r1 = min(n, r0 + per);
  int loc = 0;
  for (int r = r0; r < r1; ++r) loc += a[r];
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += u;
  }
  int run = incl - loc;
  for (int r = r0; r < r1; ++r) {
    const int v = a[r];
    a[r] = run;
    run += v;
  }
  const int total = __shfl_sync(kFull, incl, 31);
  __syncwarp();
  return total;
}

// deterministic sum of a[0..n) (smem) by one warp: 32-wide xor trees per tile, tiles in order
__device__ __forceinline__ double warp_det_sum(const double* a, int n, int lane) {
  double s = 0.0;
  for (int t = 0; t < n; t += 32) {
    double v = (t + lane < n) ? a[t + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    s += v;
  }
  return s;
}

// ---------------------------------------------------------------------------------------------
// select_layer: A3-A6 for `layer`.  mode kSelFull: single rank (or LOCAL cost scope);
// kSelLocal: A3 + local sort, pack the exchange record; kSelGlobal: merge gathered records,
// A5 on the global list, commit own requests.
// Latency-oriented: per-candidate work is spread over all NT threads; warp 0 runs the per-request
// bookkeeping and the A5 scan (lane-contiguous chunks, so the fp64 prefix is a function of the
// list length only); 7 block barriers in total.
// ---------------------------------------------------------------------------------------------
// wait_rows(L, crec): runs after the prefetch; returns true if it has itself staged the layer's
// candidate records in crec[] and each row's request in L.rreq[] (the persistent step kernel's
// row merge), false if the records are to be read from P.cand / P.cand_rs
struct NoWait {
  __device__ bool operator()(SelLayout&, int4*) const { return false; }
};
// pub(R_next): one thread publishes the next frontier (written and fenced by the caller's barrier
// or __syncwarp); the per-layer kernels release P.fr_ready[layer].  pub.entry(pos, r, node) is
// called for every frontier entry as it is written (the step kernel also writes a tagged copy).
struct PubReady {
  int* flag;
  __device__ void operator()(int) const { publish_flag(flag); }
  __device__ void entry(int, int, int) const {}
};

// bits [lo, hi) of 32-bit word w of a candidate bitmap, for the candidate range [lo, hi)
__device__ __forceinline__ unsigned word_range(int lo, int hi, int w) {
  const int a = min(max(lo - 32 * w, 0), 32), b = min(max(hi - 32 * w, 0), 32);
  const unsigned hm = b >= 32 ? ~0u : ((1u << b) - 1u);
  const unsigned lm = a >= 32 ? ~0u : ((1u << a) - 1u);
  return hm & ~lm;
}

// ---------------------------------------------------------------------------------------------
// select_tiny: A3-A6 of a small layer (<= kTinyCand candidates, <= 32 requests; NODE_SUM with
// PREFIX or FROZEN, one rank) by one warp, two candidates per lane (q = lane, lane + 32), without
// block barriers.  Same decisions and the same floating-point association as select_layer's
// block path: within-request rank by (b desc, c asc) and eligibility rank < e_r (A3), the rank of
// each eligible key among the eligible keys (A4), the tile up-scan fp64 prefix and the first
// failing entry (A5, Eq.(16)), admitted counts / offsets / node indices by ballots over the
// request's candidate range, E_r += admitted cum in canonical order, the same xor-tree totals and
// the same argmax_j reduction.  Called after select_layer's B2 (state, e_r bases, benefits staged).
// ---------------------------------------------------------------------------------------------
constexpr int kTinyCand = 64;
template <class GetCand, class Pub>
__device__ __forceinline__ void select_tiny(const Params& P, int layer, const SelLayout& L, int R, int ne, long long N0,
                                            double E0, GetCand get_cand, Pub pub) {
  const int lane = threadIdx.x & 31;
  const int k = P.k, bl = P.b_loc, nct = R * k, npar = layer & 1;
  const size_t lbase = (size_t)(layer - 1) * P.cap_rows * k;
  DevTrace& tr = P.trace[layer - 1];
  const int bc = (P.cost_scope == SMART_COST_LOCAL) ? bl : P.b_glob;
  auto sp = [&](double E, int j) {
    const double C = L.ctab[j];
    return C > 0.0 ? P.c_T * ((double)P.omega * bc + E) / C : 0.0;
  };
  const double ac = P.alpha * P.c_T;
  const double rhs0 = P.c_T * ((double)P.omega * bc + E0);
  const double dc0 = L.dtab[0];
  auto rule_ok = [&](double bj, double before, int j) {  // Eq.(16), as select_layer
    if (P.selection == SMART_FROZEN)
      return (L.ctab[0] > 0.0) ? (ac * bj * L.ctab[0] > rhs0 * dc0) : (bj > 0.0);
    const double C = L.ctab[j];
    return (C > 0.0) ? (ac * bj * C > (rhs0 + P.c_T * before) * L.dtab[j]) : (bj > 0.0);
  };
  const int nw = nct > 32 ? 2 : 1;  // candidate words in use (warp-uniform)
  // ---- A3: request, benefit, within-request rank, eligible key ----
  int rq[2], s0q[2];
  float bq[2];
  bool el[2];
  unsigned long long key[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int q = lane + 32 * i;
    rq[i] = 0;
    s0q[i] = 0;
    bq[i] = 0.f;
    el[i] = false;
    key[i] = ~0ull;
    if (q < nct) {
      const int r = L.rreq[q / k];
      const int s0 = L.off[r] * k, s1 = s0 + L.cnt[r] * k;
      const int e_r = (r + 1 < bl ? L.base[r + 1] : ne) - L.base[r];
      const float b = L.cb[q];
      int rank = 0;
#pragma unroll 8
      for (int j = s0; j < s1; ++j) {
        const float bj = L.cb[j];
        rank += (bj > b) || (bj == b && j < q);
      }
      rq[i] = r;
      s0q[i] = s0;
      bq[i] = b;
      if (rank < e_r) {
        el[i] = true;
        key[i] = sel_key(b, P.b_off + r, q - s0);
      }
    }
  }
  stamp(P, lane == 0, 11);
  // ---- A4: eligible keys compacted (ballot order), then each key's rank among them ----
  const unsigned e0 = __ballot_sync(kFull, el[0]), e1 = __ballot_sync(kFull, el[1]);
  const unsigned below = (1u << lane) - 1u;
  if (el[0]) L.keys[__popc(e0 & below)] = key[0];
  if (el[1]) L.keys[__popc(e0) + __popc(e1 & below)] = key[1];
  __syncwarp();
  int g0 = 0, g1 = 0;
#pragma unroll 8
  for (int j = 0; j < ne; ++j) {
    const unsigned long long kj = L.keys[j];  // broadcast
    g0 += kj < key[0];
    g1 += kj < key[1];
  }
  __syncwarp();
  if (el[0]) L.keys2[g0] = key[0];
  if (el[1]) L.keys2[g1] = key[1];
  __syncwarp();
  stamp(P, lane == 0, 12);
  // ---- A5: tile up-scans, tile 1 after tile 0's total; the first failing entry ----
  double bj[2], before[2];
  double t0tot = 0.0;
  unsigned fail[2] = {0u, 0u};
  before[1] = bj[1] = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (i >= nw) break;
    const int j = lane + 32 * i;
    const bool act = j < ne;
    bj[i] = act ? (double)sel_key_b(L.keys2[j]) : 0.0;
    double incl = bj[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += u;
    }
    double excl = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) excl = 0.0;
    double bf = 0.0;
    if (i == 1) bf += t0tot;
    bf += excl;
    before[i] = bf;
    if (i == 0) t0tot = __shfl_sync(kFull, incl, 31);
    fail[i] = __ballot_sync(kFull, act && !rule_ok(bj[i], bf, j));
  }
  const int js = fail[0] ? __ffs(fail[0]) - 1 : fail[1] ? 32 + __ffs(fail[1]) - 1 : ne;
  stamp(P, lane == 0, 13);
  stamp(P, lane == 0, 15);
  stamp(P, lane == 0, 16);
  // ---- A6: admitted bitmaps, per-request counts and next-frontier offsets ----
  const bool adm0 = el[0] && g0 < js, adm1 = el[1] && g1 < js;
  const unsigned a0 = __ballot_sync(kFull, adm0), a1 = __ballot_sync(kFull, adm1);
  int nx = 0, a = 0, rs0 = 0, rs1 = 0;
  if (lane < bl) {
    rs0 = L.off[lane] * k;
    rs1 = rs0 + L.cnt[lane] * k;
    a = __popc(a0 & word_range(rs0, rs1, 0)) + __popc(a1 & word_range(rs0, rs1, 1));
    nx = (L.fin[lane] || a == 0 || L.nd[lane] + a >= P.B) ? 0 : a;  // Alg.1 line 10
  }
  int incl = nx;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  const int bnext = incl - nx, tot = __shfl_sync(kFull, incl, 31);
  stamp(P, lane == 0, 17);
  // node index of an admitted candidate = admitted candidates of its request before it
  int idx[2], nxr[2], bnr[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int q = lane + 32 * i;
    idx[i] = __popc(a0 & word_range(s0q[i], q, 0)) + __popc(a1 & word_range(s0q[i], q, 1));
    nxr[i] = __shfl_sync(kFull, nx, rq[i] & 31);
    bnr[i] = __shfl_sync(kFull, bnext, rq[i] & 31);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if ((i == 0 ? adm0 : adm1) && nxr[i] > 0) {
      const int r = rq[i], pos = bnr[i] + idx[i], node = L.nd[r] + 1 + idx[i];
      P.fr[npar][pos] = make_int2(r, node);
      pub.entry(pos, r, node);
      P.fr_cum[npar][pos] = bq[i];  // NODE_SUM: b == cum
    }
  }
  if (lane < bl) P.fr_off[npar][lane] = bnext;
  if (lane == 31) *P.fr_total[npar] = incl;
  __syncwarp();
  stamp(P, lane == 0, 18);
  if (lane == 0) pub(tot);
  stamp(P, lane == 0, 19);
  // ---- after the flag: state the next layer's streaming CTAs do not read ----
  if (lane < bl) P.fr_cnt[npar][lane] = nx;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int q = lane + 32 * i;
    const bool ad = i == 0 ? adm0 : adm1;
    if (q < nct) P.cand_adm[lbase + q] = ad ? 1 : 0;
    if (ad) {
      const Cand cd = get_cand(q);
      const int r = rq[i], node = L.nd[r] + 1 + idx[i];
      const size_t o = (size_t)r * P.T + node;
      P.cand_node[lbase + q] = node;
      P.tok[o] = cd.tok;
      P.parent[o] = cd.parent;
      P.depth[o] = layer;
      P.p[o] = cd.p;
      P.cum[o] = cd.cum;
    }
  }
  stamp(P, lane == 0, 14);
  if (lane < bl) {
    if ((L.fin[lane] || a == 0 || L.nd[lane] + a >= P.B) && L.cnt[lane] > 0) P.finished[lane] = 1;
    P.n_nodes[lane] = L.nd[lane] + 1 + a;
    if (a > 0) {
      double esum = 0.0;  // canonical order (ascending candidate index)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        unsigned bits = (w == 0 ? a0 : a1) & word_range(rs0, rs1, w);
        while (bits) {
          esum += (double)L.cb[w * 32 + __ffs(bits) - 1];
          bits &= bits - 1u;
        }
      }
      L.E[lane] += esum;  // node sum (Q11)
      P.E_r[lane] = L.E[lane];
    }
  }
  __syncwarp();
  const double Ea = warp_det_sum(L.E, bl, lane);
  // trace: argmax_j S_j from the kept prefixes (same association as select_layer)
  double bestS = sp(E0, 0);
  int bestj = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int j = lane + 32 * i;
    if (j < ne) {
      const double Sa = sp(E0 + before[i] + bj[i], j + 1);
      if (Sa > bestS || (Sa == bestS && j + 1 < bestj)) {
        bestS = Sa;
        bestj = j + 1;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double os = __shfl_xor_sync(kFull, bestS, o);
    const int oj = __shfl_xor_sync(kFull, bestj, o);
    if (os > bestS || (os == bestS && oj < bestj)) {
      bestS = os;
      bestj = oj;
    }
  }
  if (lane == 0) {
    tr.S_after = sp(Ea, js) / bc;
    *P.N_glob = (int)(N0 + js);
    *P.E_glob = Ea;
    tr.executed = R > 0 ? 1 : 0;
    tr.n_rows = R;
    tr.n_cand = nct;
    tr.n_elig = ne;
    tr.n_admit = js;
    tr.argmax_j = bestj;
    tr.N0 = (int)N0;
    tr.E0 = E0;
    tr.S0 = sp(E0, 0) / bc;
    tr.dc0 = dc0;
    tr.saturated = (N0 + ne >= P.sat_from) ? 1 : 0;
    if (tr.saturated) atomicOr(P.err, kErrSaturated);
  }
  stamp(P, lane == 0, 22);
}

__device__ __forceinline__ Cand load_cand(const Cand* p) {  // L2 (written by other CTAs)
  const int4 v = __ldcg(reinterpret_cast<const int4*>(p));
  Cand c;
  c.tok = v.x;
  c.p = __int_as_float(v.y);
  c.cum = __int_as_float(v.z);
  c.parent = v.w;
  return c;
}

// ---------------------------------------------------------------------------------------------
// select_layer: A3-A6 for `layer`.  mode kSelFull: single rank (or LOCAL cost scope);
// kSelLocal: A3 + local sort, pack the exchange record; kSelGlobal: merge gathered records,
// A5 on the global list, commit own requests.
// `wait_rows` runs after the prefetch phase (per-request state, cost window, A3, E0) and before
// the layer's candidates are read: the fused layer kernel's select CTA waits there for the rows.
// Scales with the batch: per candidate only the benefit is staged, per-request admit bitmaps
// replace per-candidate flags, and every per-candidate / per-request step is spread over all NT
// threads; warp 0 runs the A5 scan (lane-contiguous chunks: the fp64 prefix is a function of
// the list length only, so any sharding reproduces it bit for bit).
// ---------------------------------------------------------------------------------------------
template <int NT, class Wait, class Pub>
__device__ void select_layer(const Params& P, int layer, int mode, char* smem, Wait wait_rows, Pub pub) {
  __shared__ SelScratch ss;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1, npar = layer & 1;
  const int k = P.k, bl = P.b_loc;
  const int b_all = (mode == kSelGlobal) ? P.b_glob : bl;
  const size_t lbase = (size_t)(layer - 1) * P.cap_rows * k;
  const bool base = (P.selection == SMART_BASELINE);  // NEXT #3 two-stage baseline (Q32)
  const bool pmean = (P.accept_model == SMART_PATH_MEAN) && !base;
  DevTrace& tr = P.trace[layer - 1];
  const int R = *P.fr_total[par];
  const int nct = R * k;  // candidates of this layer (local)
  SelLayout L = sel_layout(smem, bl, P.cap_rows * k, k, P.sort_cap);
  L.keys = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<char*>(L.E) + sel_align((size_t)b_all * 8));
  L.keys2 = L.keys + P.sort_cap;
  // optional staging of the layer's candidate records (when the scratch has room, P.sel_rec)
  unsigned long long* const kbase = L.keys;  // keys | keys2 | staged records | sort buckets
  int4* const crec = P.sel_rec ? reinterpret_cast<int4*>(L.keys + 2 * (size_t)P.sort_cap) : nullptr;
  auto get_cand = [&](int q) {
    if (crec) {
      const int4 v = crec[q];
      Cand c;
      c.tok = v.x;
      c.p = __int_as_float(v.y);
      c.cum = __int_as_float(v.z);
      c.parent = v.w;
      return c;
    }
    return load_cand(&P.cand[lbase + q]);
  };
  const int nbw = L.nbw, wf = L.wf;
  stamp(P, tid == 0, 9);

  // ---- prefetch: per-request state, the cost window, gathered records (global mode) ----
  for (int r = tid; r < bl; r += NT) {
    L.cnt[r] = P.fr_cnt[par][r];
    L.off[r] = P.fr_off[par][r];
    L.nd[r] = P.n_nodes[r] - 1;
    L.D[r] = pmean ? (float)P.leaf_cnt[r] : 1.f;  // Eq.(13), Q6
    L.fin[r] = P.finished[r];
    if (mode != kSelGlobal) L.E[r] = P.E_r[r];
  }
  for (int i = tid; i < bl * nbw; i += NT) L.bm[i] = 0u;
  {
    // cost window from N0 = drafted nodes before the layer; entries [0, max eligible + 1]
    const long long n0g = *P.N_glob;
    const int ncw = min(mode == kSelGlobal ? P.nranks * P.m_cap : nct, P.sort_cap) + 2;
    for (int j = tid; j < ncw; j += NT) {
      const long long N = min(n0g + j, (long long)P.n_cost - 1);
      L.ctab[j] = P.cost_tab[N];
      L.dtab[j] = P.dc_tab[N];
    }
  }
  if (mode == kSelGlobal) {
    for (int i = tid; i < P.nranks * P.m_cap; i += NT) {
      const int g = i / P.m_cap, e = i - g * P.m_cap;
      L.keys[i] = reinterpret_cast<const unsigned long long*>(P.xr + (size_t)g * P.xstride)[e];
    }
    for (int i = tid; i < P.b_glob; i += NT) {
      const int g = i / bl, r = i - g * bl;
      L.E[i] = reinterpret_cast<const double*>(P.xr + (size_t)g * P.xstride + (size_t)P.m_cap * 8)[r];
    }
  }
  blk_sync<NT>();  // B1

  // ---- A3 (warp 0): e_r = min(B - n_r, W, |U_r|), eligible bases; E0 (warp 1) ----
  if (warp == 0) {
    long long nl = 0;
    for (int r = lane; r < bl; r += 32) {
      int q = base ? P.Wq : P.B - L.nd[r];  // the baseline expands W per layer, no budget
      if (q > P.Wq) q = P.Wq;
      if (q < 0) q = 0;
      L.base[r] = min(q, L.cnt[r] * k);
      nl += L.nd[r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nl += __shfl_xor_sync(kFull, nl, o);
    __syncwarp();
    const int tot = warp_excl_scan_smem(L.base, bl, lane);
    if (lane == 0) {
      ss.bcast_i[2] = tot;
      ss.bcast_l[1] = nl;
    }
  } else if (warp == 1) {
    const double E0p = warp_det_sum(L.E, b_all, lane);  // global request order (Q13)
    if (lane == 0) ss.bcast_d[2] = E0p;
  }

  // ---- the layer's candidates (after the row merges): benefits b = cum / D_r (Eq.(13)) ----
  if (wait_rows(L, crec)) {  // records and row requests already staged (crec, L.rreq); the
                             // caller copies L.cb to P.cand_b after the frontier is published
    for (int q = tid; q < nct; q += NT) {
      const float cum = __int_as_float(crec[q].z);
      const float D = L.D[L.rreq[q / k]];
      L.cb[q] = (D == 1.f) ? cum : __fdiv_rn(cum, D);
    }
  } else {
    for (int q = tid; q < nct; q += NT) {
      const int r = __ldcg(&P.cand_rs[(size_t)(layer - 1) * P.cap_rows + q / k]).x;
      const int4 rec = __ldcg(reinterpret_cast<const int4*>(&P.cand[lbase + q]));  // whole record
      const float cum = __int_as_float(rec.z);
      if (crec) crec[q] = rec;  // staged for the commit (no second L2 round trip)
      const float D = L.D[r];
      const float b = (D == 1.f) ? cum : __fdiv_rn(cum, D);
      L.cb[q] = b;
      P.cand_b[lbase + q] = b;
      if (q % k == 0) L.rreq[q / k] = r;
    }
  }
  blk_sync<NT>();  // B2
  stamp(P, tid == 0, 10);
  int ne = ss.bcast_i[2];
  long long N0 = ss.bcast_l[1];
  if (mode == kSelFull && !base && !pmean && nct <= kTinyCand && bl <= 32) {
    // small layer: the rest by warp 0 alone (the caller's next barrier waits for it)
    if (warp == 0) select_tiny(P, layer, L, R, ne, N0, ss.bcast_d[2], get_cand, pub);
    return;
  }
  if (mode != kSelGlobal) {
    // within-request rank by (b desc, c asc); eligible if rank < e_r (early exit past e_r)
    for (int q = tid; q < nct; q += NT) {
      const int r = L.rreq[q / k];
      const int s0 = L.off[r] * k, s1 = s0 + L.cnt[r] * k;
      const int e_r = (r + 1 < bl ? L.base[r + 1] : ne) - L.base[r];
      const float b = L.cb[q];
      int rank = 0;
#pragma unroll 4
      for (int j = s0; j < s1; ++j) {  // no early exit: uniform trip counts, pipelined loads
        const float bj = L.cb[j];
        rank += (bj > b) || (bj == b && j < q);
      }
      if (rank < e_r) L.keys[L.base[r] + rank] = sel_key(b, P.b_off + r, q - s0);
    }
    blk_sync<NT>();  // B3
  }
  stamp(P, tid == 0, 11);

  // ---- A4: sort (local list, or the gathered lists of all ranks) ----
  const int nsort = base ? 0 : (mode == kSelGlobal) ? P.nranks * P.m_cap : ne;
  if (base) {
    // the baseline admits every eligible candidate: no global order, no rule (Q32)
  } else if (nsort <= 256) {
    // rank sort (keys unique; padding ~0 keys sort to the end); two keys per shared load
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(L.keys);
    for (int i = tid; i < nsort; i += NT) {
      const unsigned long long key = L.keys[i];
      int r0 = 0, r1 = 0;
      int f = 0;
#pragma unroll 4
      for (; f + 1 < nsort; f += 2) {
        const ulonglong2 v = k2[f >> 1];
        r0 += (v.x < key);
        r1 += (v.y < key);
      }
      if (f < nsort) r0 += (L.keys[f] < key);
      L.keys2[r0 + r1] = key;
    }
    blk_sync<NT>();  // B4
    unsigned long long* t = L.keys;
    L.keys = L.keys2;
    L.keys2 = t;
  } else {
    // long lists: bucket pass on the key's top 12 bits (benefit sign/exponent/3 mantissa bits,
    // order-preserving), then each key's rank inside its bucket; keys are unique, so the result
    // is exactly the sorted order (the bitonic network cost ~470 cycles per stage, 66 stages)
    int* bcnt = reinterpret_cast<int*>(kbase + 2 * (size_t)P.sort_cap +
                                       (P.sel_rec ? (size_t)P.cap_rows * P.k * 2 : 0));  // counts -> cursors
    int* boff = bcnt + kSortBuckets;        // [kSortBuckets] exclusive offsets
    for (int i = tid; i < kSortBuckets; i += NT) bcnt[i] = 0;
    blk_sync<NT>();
    for (int i = tid; i < nsort; i += NT) atomicAdd(&bcnt[(int)(L.keys[i] >> (64 - kSortBucketBits))], 1);
    blk_sync<NT>();
    for (int i = tid; i < kSortBuckets; i += NT) boff[i] = bcnt[i];
    blk_sync<NT>();
    excl_scan_int<NT>(boff, kSortBuckets, ss);
    for (int i = tid; i < kSortBuckets; i += NT) bcnt[i] = boff[i];
    blk_sync<NT>();
    for (int i = tid; i < nsort; i += NT) {
      const unsigned long long key = L.keys[i];
      L.keys2[atomicAdd(&bcnt[(int)(key >> (64 - kSortBucketBits))], 1)] = key;
    }
    blk_sync<NT>();
    for (int p = tid; p < nsort; p += NT) {
      const unsigned long long key = L.keys2[p];
      const int bk = (int)(key >> (64 - kSortBucketBits));
      const int b0 = boff[bk], b1 = bcnt[bk];  // the bucket's range in keys2
      int rank = b0;
      for (int q = b0; q < b1; ++q) rank += (L.keys2[q] < key);
      L.keys[rank] = key;
    }
    blk_sync<NT>();
  }
  stamp(P, tid == 0, 12);

  if (mode == kSelLocal) {
    unsigned long long* xk = reinterpret_cast<unsigned long long*>(P.xs);
    double* xE = reinterpret_cast<double*>(P.xs + (size_t)P.m_cap * 8);
    int* xh = reinterpret_cast<int*>(P.xs + (size_t)P.m_cap * 8 + (size_t)bl * 8);
    for (int i = tid; i < P.m_cap; i += NT) xk[i] = i < ne ? L.keys[i] : ~0ull;
    for (int r = tid; r < bl; r += NT) {
      xh[r] = L.nd[r];
      xE[r] = L.E[r];
    }
    if (tid == 0) {
      xh[bl] = ne;
      xh[bl + 1] = R;
    }
    return;
  }

  const int bc = (P.cost_scope == SMART_COST_LOCAL) ? bl : P.b_glob;
  auto sp = [&](double E, int j) {  // b*S at N0 + j from the prefetched window
    const double C = L.ctab[j];
    return C > 0.0 ? P.c_T * ((double)P.omega * bc + E) / C : 0.0;
  };
  // ---- A5 (warp 0): Eq.(16) scan over the sorted list -> the cut js (the only result the
  // commit waits for); argmax_j S_j and the admitted benefit sum are computed by warp 1 during
  // the commit's tail (a5_report below) ----
  if (mode == kSelGlobal && warp == 0) {
    long long nloc = 0, eloc = 0, rloc = 0;
    for (int i = lane; i < P.b_glob; i += 32) {
      const int g = i / bl, r = i - g * bl;
      nloc += reinterpret_cast<const int*>(P.xr + (size_t)g * P.xstride + (size_t)P.m_cap * 8 + (size_t)bl * 8)[r];
    }
    for (int g = lane; g < P.nranks; g += 32) {
      const int* h = reinterpret_cast<const int*>(P.xr + (size_t)g * P.xstride + (size_t)P.m_cap * 8 + (size_t)bl * 8);
      eloc += h[bl];
      rloc += h[bl + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nloc += __shfl_xor_sync(kFull, nloc, o);
      eloc += __shfl_xor_sync(kFull, eloc, o);
      rloc += __shfl_xor_sync(kFull, rloc, o);
    }
    if (lane == 0) {
      ss.bcast_l[1] = nloc;
      ss.bcast_i[2] = (int)eloc;
      ss.bcast_i[4] = (int)rloc;
    }
    __syncwarp();
  }
  const double E0 = ss.bcast_d[2];  // precomputed before the wait
  const double ac = P.alpha * P.c_T;
  const double rhs0 = P.c_T * ((double)P.omega * bc + E0);
  const double dc0 = L.dtab[0];
  if (mode == kSelGlobal) {
    blk_sync<NT>();
    N0 = ss.bcast_l[1];
    ne = ss.bcast_i[2];
  }
  // lists longer than kA5Par: the looped form of the short-list scan below (same association,
  // a function of the entry index only)
  const bool big = !base && ne > kA5Par;
  auto rule_ok = [&](double bj, double before, int j) {
    // Eq.(16), strict: alpha*c_T*b/dc > c_T*(omega*b + E)/cost, cross-multiplied (dc, cost > 0;
    // cost == 0 means S := 0, i.e. admit any positive benefit)
    if (P.selection == SMART_FROZEN)
      return (L.ctab[0] > 0.0) ? (ac * bj * L.ctab[0] > rhs0 * dc0) : (bj > 0.0);
    const double C = L.ctab[j];
    return (C > 0.0) ? (ac * bj * C > (rhs0 + P.c_T * before) * L.dtab[j]) : (bj > 0.0);
  };
  if (big) {
    // long lists: fp64 prefix = 32-wide up-scan inside each tile of 32 entries plus the
    // exclusive prefix of the tile totals (lane-contiguous groups of tiles, then a warp
    // up-scan: a function of the list length only); the cut is the smallest failing index
    // (ballot per tile, shared min)
    double* scr = reinterpret_cast<double*>(L.keys2);
    const int ntile = (ne + 31) / 32;  // <= 128 (tile_d holds 260)
    if (tid == 0) ss.bcast_i[3] = ne;
    for (int t = warp; t < ntile; t += NT / 32) {
      const int j = t * 32 + lane;
      const double bj = j < ne ? (double)sel_key_b(L.keys[j]) : 0.0;
      double incl = bj;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += u;
      }
      double excl = __shfl_up_sync(kFull, incl, 1);
      if (lane == 0) excl = 0.0;
      if (j < ne) scr[j] = excl;
      if (lane == 31) ss.tile_d[t] = incl;
    }
    blk_sync<NT>();
    if (warp == 0) {  // tile totals -> exclusive prefixes: lane-contiguous groups, warp up-scan
      const int per = (ntile + 31) >> 5;
      const int t0 = min(ntile, lane * per), t1 = min(ntile, t0 + per);
      double loc = 0.0;
      for (int t = t0; t < t1; ++t) loc += ss.tile_d[t];
      double inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += u;
      }
      double run = __shfl_up_sync(kFull, inc, 1);
      if (lane == 0) run = 0.0;
      for (int t = t0; t < t1; ++t) {
        const double v = ss.tile_d[t];
        ss.tile_d[t] = run;
        run += v;
      }
    }
    blk_sync<NT>();
    for (int t = warp; t < ntile; t += NT / 32) {
      const int j = t * 32 + lane;
      bool fail = false;
      if (j < ne) {
        const double before = ss.tile_d[t] + scr[j];
        scr[j] = before;
        fail = !rule_ok((double)sel_key_b(L.keys[j]), before, j);
      }
      const unsigned bal = __ballot_sync(kFull, fail);
      if (bal && lane == 0) atomicMin(&ss.bcast_i[3], t * 32 + __ffs(bal) - 1);
    }
    blk_sync<NT>();
    if (tid == 0) {
      ss.bcast_i[5] = ne;
      ss.bcast_i[6] = -2;  // argmax_j from the kept prefixes, in the tail
      ss.bcast_l[0] = N0;
    }
  } else if (base) {
    if (tid == 0) {
      ss.bcast_i[3] = ne;  // all eligible admitted
      ss.bcast_i[5] = ne;
      ss.bcast_i[6] = 0;
      ss.bcast_l[0] = N0;
    }
  } else if (ne <= kA5Par) {
    // short lists: one entry per thread.  fp64 prefix = 32-wide up-scan inside each tile of 32
    // entries plus the preceding tiles' totals in order (a function of the entry index only, so
    // any block size and any sharding give the same bits); the cut is the first failing entry
    // (ballots, then a warp min).  The prefixes are kept in the sort scratch so that the trace's
    // argmax_j S_j is computed after the next frontier is published (off the critical path).
    const int j = tid;
    const bool act = j < ne;
    const double bj = act ? (double)sel_key_b(L.keys[j]) : 0.0;
    double incl = bj;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += u;
    }
    double excl = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) excl = 0.0;
    if (lane == 31 && tid < kA5Par) ss.tile_d[warp] = incl;
    blk_sync<NT>();
    if (tid < kA5Par) {
      // preceding tiles' totals in order (the loads issued together, the adds predicated)
      double tv[kA5Par / 32];
#pragma unroll
      for (int w = 0; w < kA5Par / 32; ++w) tv[w] = ss.tile_d[w];
      double before = 0.0;
#pragma unroll
      for (int w = 0; w < kA5Par / 32; ++w)
        if (w < warp) before += tv[w];
      before += excl;
      if (act) reinterpret_cast<double*>(L.keys2)[j] = before;
      const unsigned bal = __ballot_sync(kFull, act && !rule_ok(bj, before, j));
      if (lane == 0) ss.wred_i[warp] = bal ? warp * 32 + __ffs(bal) - 1 : ne;
    }
    blk_sync<NT>();
    if (warp == 0) {
      const int js0 = (int)__reduce_min_sync(kFull, (unsigned)(lane < (ne + 31) / 32 ? ss.wred_i[lane] : ne));
      if (lane == 0) {
        ss.bcast_i[3] = js0;
        ss.bcast_i[5] = ne;
        ss.bcast_i[6] = -2;  // argmax_j from the kept prefixes, in the tail
        ss.bcast_l[0] = N0;
      }
    }
  } else if (warp == 0) {
    // lane-contiguous chunks: sequential fp64 prefix inside a lane, warp scan of lane totals
    const int per = (ne + 31) >> 5;
    const int j0 = min(ne, lane * per), j1 = min(ne, j0 + per);
    double lt = 0.0;
    for (int j = j0; j < j1; ++j) lt += (double)sel_key_b(L.keys[j]);
    double lex = lt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(kFull, lex, o);
      if (lane >= o) lex += u;
    }
    lex -= lt;
    int first_fail = ne;
    double before = lex;
    for (int j = j0; j < j1; ++j) {
      const double bj = (double)sel_key_b(L.keys[j]);
      if (!rule_ok(bj, before, j)) {
        first_fail = j;
        break;
      }
      before += bj;
    }
    first_fail = __reduce_min_sync(kFull, first_fail);
    if (lane == 0) {
      ss.bcast_i[3] = first_fail;
      ss.bcast_i[5] = ne;
      ss.bcast_i[6] = -1;  // argmax_j computed by warp 1 in the tail
      ss.bcast_l[0] = N0;
    }
  }
  blk_sync<NT>();  // B5
  const int js = ss.bcast_i[3];
  stamp(P, tid == 0, 13);

  // ---- A6: commit (own requests) ----
  // (1) admit bitmaps (bit c of request r <=> candidate c = slot * k + rank admitted); the
  // admitted records (and parent path sums) are fetched here so their latency hides behind B6
  constexpr int kPre = 4;
  Cand cdr[kPre];
  double ppr[kPre];
  int qr[kPre];
#pragma unroll
  for (int it = 0; it < kPre; ++it) qr[it] = -1;
  // NODE_SUM with <= 32 requests: warp 0 runs the per-request step (3) right after the bitmaps
  // (E from the staged benefits, b == cum) while warps 1.. write the nodes
  const bool fast3 = (bl <= 32) && !pmean;
  const int c0t = fast3 ? 32 : 0, cstep = fast3 ? NT - 32 : NT;
  for (int j = tid - c0t, it = 0; j < js && tid >= c0t; j += cstep, ++it) {
    const unsigned long long key = L.keys[j];
    const int r = sel_key_r(key) - P.b_off;
    if (r < 0 || r >= bl) continue;
    const int c = sel_key_c(key);
    atomicOr(&L.bm[r * nbw + (c >> 5)], 1u << (c & 31));
#pragma unroll
    for (int u = 0; u < kPre; ++u)
      if (u == it) {
        qr[u] = L.off[r] * k + c;
        cdr[u] = get_cand(qr[u]);
      }
  }
  if (pmean) {
#pragma unroll
    for (int u = 0; u < kPre; ++u)
      if (qr[u] >= 0) ppr[u] = P.path_sum[(size_t)L.rreq[qr[u] / k] * P.T + cdr[u].parent];
  }
  stamp(P, tid == 0, 15);
  blk_sync<NT>();  // B6
  stamp(P, tid == 0, 16);
  auto bits_below = [&](int r, int c) {  // admitted candidates of r with index < c
    int n = 0;
    for (int w = 0; w < (c >> 5); ++w) n += __popc(L.bm[r * nbw + w]);
    if (c & 31) n += __popc(L.bm[r * nbw + (c >> 5)] & ((1u << (c & 31)) - 1u));
    return n;
  };
  // The next frontier depends on the bitmaps only, so it is built and published first (the
  // next layer kernel's streaming CTAs start on the flag); node records, E and the trace follow.
  // (3a) per request: admitted count, finish, next-frontier count and offsets.  Up to 32 requests:
  // warp 0 alone, scan by shuffles; else all threads + block scan.
  const bool one_warp = bl <= 32;
  auto finished_r = [&](int r, int a) {  // Alg.1 line 10
    return L.fin[r] || a == 0 || (!base && L.nd[r] + a >= P.B);
  };
  if (one_warp) {
    // warp 0 alone: counts, offsets and the admitted candidates' frontier entries, then the
    // flag (no block barrier on this path; the fence covers only warp 0's few stores)
    if (warp == 0) {
      int nx = 0;
      if (lane < bl) {
        int a = 0;
        for (int w = 0; w < nbw; ++w) a += __popc(L.bm[lane * nbw + w]);
        L.adm[lane] = a;
        nx = finished_r(lane, a) ? 0 : a;
        L.nxt[lane] = nx;
      }
      stamp(P, tid == 0, 20);
      int incl = nx;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      stamp(P, tid == 0, 21);
      if (lane < bl) L.base[lane] = incl - nx;
      __syncwarp();
      stamp(P, tid == 0, 17);
      for (int j = lane; j < js; j += 32) {
        const unsigned long long key = L.keys[j];
        const int r = sel_key_r(key) - P.b_off;
        if (r < 0 || r >= bl || L.nxt[r] == 0) continue;
        const int c = sel_key_c(key);
        const int q = L.off[r] * k + c;
        const int idx = bits_below(r, c);
        P.fr[npar][L.base[r] + idx] = make_int2(r, L.nd[r] + 1 + idx);
        pub.entry(L.base[r] + idx, r, L.nd[r] + 1 + idx);
        P.fr_cum[npar][L.base[r] + idx] = pmean ? get_cand(q).cum : L.cb[q];  // NODE_SUM: b == cum
      }
      if (lane < bl) P.fr_off[npar][lane] = incl - nx;
      if (lane == 31) *P.fr_total[npar] = incl;
      const int tot = __shfl_sync(kFull, incl, 31);
      __syncwarp();
      stamp(P, tid == 0, 18);
      if (lane == 0) pub(tot);
      stamp(P, tid == 0, 19);
    }
    blk_sync<NT>();  // B7: per-request counts and offsets for everyone
  } else {
    for (int r = tid; r < bl; r += NT) {
      int a = 0;
      for (int w = 0; w < nbw; ++w) a += __popc(L.bm[r * nbw + w]);
      L.adm[r] = a;
      const int nx = finished_r(r, a) ? 0 : a;
      L.nxt[r] = nx;
      L.base[r] = nx;
    }
    blk_sync<NT>();  // B7
    const int total = excl_scan_int<NT>(L.base, bl, ss);  // next-frontier offsets
    for (int r = tid; r < bl; r += NT) P.fr_off[npar][r] = L.base[r];
    if (tid == 0) *P.fr_total[npar] = total;
    // (4) next frontier (own requests that continue), with the cum of each node for the row merge
    for (int q = tid; q < nct; q += NT) {
      const int r = L.rreq[q / k];
      const int c = q - L.off[r] * k;
      if (!((L.bm[r * nbw + (c >> 5)] >> (c & 31)) & 1u) || L.nxt[r] == 0) continue;
      const int idx = bits_below(r, c);
      P.fr[npar][L.base[r] + idx] = make_int2(r, L.nd[r] + 1 + idx);
      pub.entry(L.base[r] + idx, r, L.nd[r] + 1 + idx);
      P.fr_cum[npar][L.base[r] + idx] = pmean ? get_cand(q).cum : L.cb[q];  // NODE_SUM: b == cum
    }
    blk_sync<NT>();  // B8: the next frontier is complete
    if (tid == 0) pub(total);
  }
  // after the flag: state the next layer's streaming CTAs do not read
  for (int r = tid; r < bl; r += NT) P.fr_cnt[npar][r] = L.nxt[r];
  for (int q = tid; q < nct; q += NT) {
    const int r = L.rreq[q / k];
    const int c = q - L.off[r] * k;
    P.cand_adm[lbase + q] = (L.bm[r * nbw + (c >> 5)] >> (c & 31)) & 1u;
  }
  stamp(P, tid == 0, 14);
  // (2) admitted candidates write their node (index among the request's admits in canonical
  // order = admit bits below) and stage cum / parent path sum for (3b)
  auto commit_node = [&](int q, const Cand& cd, double pps) {
    const int r = L.rreq[q / k];
    const int c = q - L.off[r] * k;
    const int idx = bits_below(r, c);
    const int node = L.nd[r] + 1 + idx;
    const size_t o = (size_t)r * P.T + node;
    P.cand_node[lbase + q] = node;
    P.tok[o] = cd.tok;
    P.parent[o] = cd.parent;
    P.depth[o] = layer;
    P.p[o] = cd.p;
    P.cum[o] = cd.cum;
    L.cslot[r * wf + idx] = cd.cum;
    if (pmean) {
      L.pslot[r * wf + idx] = pps;
      P.path_sum[o] = pps + (double)cd.cum;
    }
  };
#pragma unroll
  for (int u = 0; u < kPre; ++u)
    if (qr[u] >= 0) commit_node(qr[u], cdr[u], pmean ? ppr[u] : 0.0);
  for (int j = tid - c0t + kPre * cstep; j < js && tid >= c0t; j += cstep) {  // beyond the register prefetch
    const unsigned long long key = L.keys[j];
    const int r = sel_key_r(key) - P.b_off;
    if (r < 0 || r >= bl) continue;
    const int q = L.off[r] * k + sel_key_c(key);
    const Cand cd = get_cand(q);
    commit_node(q, cd, pmean ? P.path_sum[(size_t)r * P.T + cd.parent] : 0.0);
  }
  if (!fast3) blk_sync<NT>();  // B9 (fast3: warp 0 needs only the staged benefits)
  // (3b) per request: finished flag, node count, E (canonical order)
  for (int r = tid; r < bl && (!one_warp || warp == 0); r += NT) {
    const int a = L.adm[r];
    if (finished_r(r, a) && L.cnt[r] > 0) P.finished[r] = 1;
    P.n_nodes[r] = L.nd[r] + 1 + a;
    if (a == 0) continue;
    const int gi = (mode == kSelGlobal ? P.b_off : 0) + r;
    if (!pmean) {
      double esum = 0.0;
      if (fast3) {  // staged benefits (b == cum), canonical order
        const int s0 = L.off[r] * k;
        for (int w = 0; w < nbw; ++w) {
          unsigned bits = L.bm[r * nbw + w];
          while (bits) {
            esum += (double)L.cb[s0 + w * 32 + __ffs(bits) - 1];
            bits &= bits - 1u;
          }
        }
      } else {
        for (int u = 0; u < a; ++u) esum += (double)L.cslot[r * wf + u];
      }
      L.E[gi] += esum;  // node sum (Q11)
    } else {
      // Eq.(2) path mean of the committed tree: leaves lose their admitted-into parents
      double psum_new = 0.0, psum_par = 0.0;
      int nparents = 0, u = 0, prev_row = -1;
      for (int w = 0; w < nbw; ++w) {
        unsigned bits = L.bm[r * nbw + w];
        while (bits) {
          const int c = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1u;
          const double pps = L.pslot[r * wf + u];
          psum_new += pps + (double)L.cslot[r * wf + u];
          if (c / k != prev_row) {  // first admitted child of this frontier row
            psum_par += pps;
            ++nparents;
            prev_row = c / k;
          }
          ++u;
        }
      }
      const int lc = P.leaf_cnt[r] - nparents + a;
      const double ls = P.leaf_sum[r] - psum_par + psum_new;
      P.leaf_cnt[r] = lc;
      P.leaf_sum[r] = ls;
      L.E[gi] = ls / (double)lc;
    }
    P.E_r[r] = L.E[gi];
  }
  if (one_warp) __syncwarp();
  else blk_sync<NT>();  // B10: E complete for the totals
  // ---- totals after the layer (trace S_after) ∥ the A5 report (argmax_j S_j, trace) ----
  if (warp == 0 && mode == kSelFull) {
    const double Ea = warp_det_sum(L.E, bl, lane);
    if (lane == 0) {
      tr.S_after = sp(Ea, js) / bc;
      *P.N_glob = (int)(ss.bcast_l[0] + js);
      *P.E_glob = Ea;
    }
  }
  const bool wide_argmax = ss.bcast_i[6] == -2 && ss.bcast_i[5] > kA5Par;
  if (wide_argmax) {
    // long lists: S_j over all threads (one fp64 division each), per-warp winners in smem
    const int ne_r = ss.bcast_i[5];
    const double* scr = reinterpret_cast<const double*>(L.keys2);
    double bestS = -1.0;
    int bestj = ne_r + 1;
    for (int j = tid; j < ne_r; j += NT) {
      const double Sa = sp(E0 + scr[j] + (double)sel_key_b(L.keys[j]), j + 1);
      if (Sa > bestS || (Sa == bestS && j + 1 < bestj)) {
        bestS = Sa;
        bestj = j + 1;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(kFull, bestS, o);
      const int oj = __shfl_xor_sync(kFull, bestj, o);
      if (os > bestS || (os == bestS && oj < bestj)) {
        bestS = os;
        bestj = oj;
      }
    }
    if (lane == 0) {
      ss.wred_d[warp] = bestS;
      ss.tile_i[warp] = bestj;
    }
    blk_sync<NT>();
  }
  if (warp == 1 && ss.bcast_i[6] == -2) {
    // short lists: S_j from the prefixes the parallel A5 kept (same association as the cut)
    const int ne_r = ss.bcast_i[5];
    const long long N0r = ss.bcast_l[0];
    const double* scr = reinterpret_cast<const double*>(L.keys2);
    double bestS = sp(E0, 0);
    int bestj = 0;
    for (int j = wide_argmax ? ne_r : lane; j < ne_r; j += 32) {
      const double Sa = sp(E0 + scr[j] + (double)sel_key_b(L.keys[j]), j + 1);
      if (Sa > bestS || (Sa == bestS && j + 1 < bestj)) {
        bestS = Sa;
        bestj = j + 1;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(kFull, bestS, o);
      const int oj = __shfl_xor_sync(kFull, bestj, o);
      if (os > bestS || (os == bestS && oj < bestj)) {
        bestS = os;
        bestj = oj;
      }
    }
    if (wide_argmax && lane == 0) {
      for (int w = 0; w < NT / 32; ++w) {  // warp winners in warp order
        const double os = ss.wred_d[w];
        const int oj = ss.tile_i[w];
        if (oj <= ne_r && (os > bestS || (os == bestS && oj < bestj))) {
          bestS = os;
          bestj = oj;
        }
      }
    }
    if (lane == 0) {
      const double ab = js < ne_r ? scr[js] : (ne_r > 0 ? scr[ne_r - 1] + (double)sel_key_b(L.keys[ne_r - 1]) : 0.0);
      const int R_all = (mode == kSelGlobal) ? ss.bcast_i[4] : R;
      tr.executed = R_all > 0 ? 1 : 0;
      tr.n_rows = R;
      tr.n_cand = nct;
      tr.n_elig = ne_r;
      tr.n_admit = js;
      tr.argmax_j = bestj;
      tr.N0 = (int)N0r;
      tr.E0 = E0;
      tr.S0 = sp(E0, 0) / bc;
      tr.dc0 = dc0;
      tr.saturated = (N0r + ne_r >= P.sat_from) ? 1 : 0;
      if (tr.saturated) atomicOr(P.err, kErrSaturated);
      if (mode != kSelFull) {
        const double Ea = E0 + ab;
        tr.S_after = sp(Ea, js) / bc;
        *P.N_glob = (int)(N0r + js);
        *P.E_glob = Ea;
      }
    }
  } else if (warp == 1) {
    const int ne_r = ss.bcast_i[5];
    const int argmax_pre = ss.bcast_i[6];  // long lists: already reduced by the A5 groups
    const long long N0r = ss.bcast_l[0];
    const int R_all = (mode == kSelGlobal) ? ss.bcast_i[4] : R;
    const double Sb0 = sp(E0, 0);
    const int per = (ne_r + 31) >> 5;
    const int j0 = min(ne_r, lane * per), j1 = min(ne_r, j0 + per);
    double lt = 0.0;
    for (int j = j0; j < j1; ++j) lt += (double)sel_key_b(L.keys[j]);
    double lex = lt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(kFull, lex, o);
      if (lane >= o) lex += u;
    }
    lex -= lt;
    double bestS = Sb0, before = lex, ab = 0.0;
    int bestj = 0;
    for (int j = j0; j < j1; ++j) {
      const double bj = (double)sel_key_b(L.keys[j]);
      if (argmax_pre < 0) {
        const double Sa = sp(E0 + before + bj, j + 1);
        if (Sa > bestS || (Sa == bestS && j + 1 < bestj)) {
          bestS = Sa;
          bestj = j + 1;
        }
      }
      if (j < js) ab += bj;
      before += bj;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(kFull, bestS, o);
      const int oj = __shfl_xor_sync(kFull, bestj, o);
      if (os > bestS || (os == bestS && oj < bestj)) {
        bestS = os;
        bestj = oj;
      }
      ab += __shfl_xor_sync(kFull, ab, o);
    }
    if (lane == 0) {
      tr.executed = R_all > 0 ? 1 : 0;
      tr.n_rows = R;
      tr.n_cand = nct;
      tr.n_elig = ne_r;
      tr.n_admit = js;
      tr.argmax_j = base ? 0 : argmax_pre >= 0 ? argmax_pre : bestj;
      tr.N0 = (int)N0r;
      tr.E0 = E0;
      tr.S0 = Sb0 / bc;
      tr.dc0 = dc0;
      tr.saturated = (N0r + ne_r >= P.sat_from) ? 1 : 0;
      if (tr.saturated) atomicOr(P.err, kErrSaturated);
      if (mode != kSelFull) {
        // NODE_SUM: E after = E0 + sum of admitted benefits (exact); PATH_MEAN: approximate
        const double Ea = E0 + ab;
        tr.S_after = sp(Ea, js) / bc;
        *P.N_glob = (int)(N0r + js);
        *P.E_glob = Ea;
      }
    }
  }
  stamp(P, tid == 0, 22);
}

}  // namespace smart
