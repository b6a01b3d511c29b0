// expand.cu — K1 `smart_expand_step`: A1 (top-k + softmax of every frontier row, P:216-222,
// P:160) and A2 (path score cum = cum(parent) * p, Eq.(3)) on B200 (sm_100a).
//
// Design:
//  * HBM-bound stream: the frontier rows are cut into 16 KiB chunks; a persistent grid of
//    (#SMs x occupancy) CTAs takes a balanced contiguous range of (row, chunk) units, so one
//    kernel serves 1 row (cfg2 layer 1) and 2304 rows (cfg5) alike.  128-bit L1-bypassing
//    loads, the next chunk prefetched into registers while the current one is reduced.
//  * softmax: each warp reduces its 1024/512 elements of a chunk to (max, sum exp) with a
//    fixed shuffle tree and writes that partial; the row merge combines the cpr x 8 partials
//    in fixed order, so Z is bit-identical for any grid size or sharding (Q24, §8e).
//  * top-k: each warp keeps a running sorted top-k list in registers (lane i = entry i,
//    k <= 32).  A segment's first chunk seeds the list with the top-k lane maxima (bitonic
//    sort of 32 keys); afterwards only lanes whose max beats the threshold scan for
//    candidates.  A CTA-wide threshold hint (64-bit atomicMax of the warps' k-th keys) cuts
//    the candidates of all 8 warps.  The union of warp lists always contains the exact top-k.
//  * the CTA that completes a row's last chunk (arrival counter) merges the partials:
//    Z, exact top-k by (value desc, index asc), p = exp(x - M)/Z, cum = cum(parent) * p.
#include "smart_internal.cuh"

namespace smart {

namespace {

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long make_key(float v, int i) {
  return ((unsigned long long)float_orderable(v) << 32) | (unsigned long long)(0xffffffffu - (unsigned)i);
}
__device__ __forceinline__ void split_key(unsigned long long key, float& v, int& i) {
  uint32_t o = (uint32_t)(key >> 32);
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  v = __uint_as_float(u);
  i = (int)(0xffffffffu - (uint32_t)(key & 0xffffffffu));
}

// insert (nv, ni) into the warp's sorted list (lane e holds entry e, e < k).
// Precondition: (nv, ni) is better than entry k-1.
__device__ __forceinline__ void warp_insert(float& lv, int& li, float nv, int ni, int k, int lane) {
  bool ahead = (lane < k) && better(lv, li, nv, ni);
  int pos = __popc(__ballot_sync(kFull, ahead));
  float uv = __shfl_up_sync(kFull, lv, 1);
  int ui = __shfl_up_sync(kFull, li, 1);
  if (lane == pos) {
    lv = nv;
    li = ni;
  } else if (lane > pos && lane < k) {
    lv = uv;
    li = ui;
  }
}

// bitonic sort of one key per lane, descending in `better` order; carries `src`.
__device__ __forceinline__ void warp_bitonic_desc(float& v, int& i, int& src, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      float ov = __shfl_xor_sync(kFull, v, stride);
      int oi = __shfl_xor_sync(kFull, i, stride);
      int os = __shfl_xor_sync(kFull, src, stride);
      bool desc_block = ((lane & size) == 0) || size == 32;
      bool lower = (lane & stride) == 0;
      bool mine = better(v, i, ov, oi);
      bool keep = (lower == desc_block) ? mine : !mine;
      if (!keep) {
        v = ov;
        i = oi;
        src = os;
      }
    }
  }
}

template <bool BF16>
struct Traits {
  static constexpr int EPV = BF16 ? 8 : 4;                  // elements per 16 B vector
  static constexpr int EPT = kVecPerThread * EPV;           // elements per thread per chunk
};

// element n (= j*EPV + e) of thread `tid` in chunk c -> row element index
template <bool BF16>
__device__ __forceinline__ int elem_index(int chunk_base, int tid, int n) {
  constexpr int EPV = Traits<BF16>::EPV;
  return chunk_base + ((n / EPV) * kStreamThreads + tid) * EPV + (n % EPV);
}

// load this thread's 4 vectors of chunk c of a row; out-of-range elements are -inf.
template <bool BF16, bool ALIGNED>
__device__ __forceinline__ void load_chunk(const char* row, int chunk_base, int V, int tid, uint4 (&raw)[kVecPerThread]) {
  constexpr int EPV = Traits<BF16>::EPV;
  constexpr int ESZ = BF16 ? 2 : 4;
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    int e0 = chunk_base + (j * kStreamThreads + tid) * EPV;
    if (ALIGNED && e0 + EPV <= V) {
      raw[j] = ldg_stream(row + (size_t)e0 * ESZ);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = BF16 ? 0xff80ff80u : 0xff800000u;  // -inf
      if (e0 < V) {
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          if (e0 + e < V) {
            if (BF16) {
              uint32_t h = *reinterpret_cast<const unsigned short*>(row + (size_t)(e0 + e) * 2);
              int q = e >> 1;
              w[q] = (e & 1) ? ((w[q] & 0x0000ffffu) | (h << 16)) : ((w[q] & 0xffff0000u) | h);
            } else {
              w[e] = *reinterpret_cast<const uint32_t*>(row + (size_t)(e0 + e) * 4);
            }
          }
        }
      }
      raw[j] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

template <bool BF16>
__device__ __forceinline__ void unpack(const uint4 (&raw)[kVecPerThread], float (&x)[Traits<BF16>::EPT]) {
#pragma unroll
  for (int j = 0; j < kVecPerThread; ++j) {
    uint32_t w[4] = {raw[j].x, raw[j].y, raw[j].z, raw[j].w};
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

// resolve the logits row of frontier row `row` (layer parity `par`)
__device__ __forceinline__ const char* row_ptr(const Params& P, int par, const char* base, long long ld_bytes,
                                              int row) {
  if (P.row_mode == SMART_ROWS_NODE) {
    int2 fe = P.fr[par][row];
    return base + ((long long)fe.x * P.T + fe.y) * ld_bytes;
  }
  return base + (long long)row * ld_bytes;
}

struct ExpandShared {
  unsigned long long tau;                       // CTA threshold hint (best k-th key)
  int last;                                     // this CTA merges the row
  int wcnt[kStreamWarps];
  float bufv[kStreamWarps][kWarpBuf];
  int bufi[kStreamWarps][kWarpBuf];
  // row merge
  float red[kStreamWarps];
  float mlv[kStreamWarps][kMaxK];
  int mli[kStreamWarps][kMaxK];
  int seg_start[256];
  int nseg;
};

// ---- row merge by the CTA that completed the row (all 256 threads) ----
__device__ void merge_row(const Params& P, int layer, int par, int row, ExpandShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = P.k, cpr = P.cpr;
  const float2* ms = P.ms + (size_t)row * cpr * kStreamWarps;
  const int npart = cpr * kStreamWarps;

  // (1) softmax normaliser: M = max, Z = sum s*exp(m - M), fixed association order
  float m = -INFINITY;
  for (int q = tid; q < npart; q += kStreamThreads) m = fmaxf(m, __ldcg(&ms[q].x));
  m = warp_max(m);
  if (lane == 0) sh.red[warp] = m;
  __syncthreads();
  float M = sh.red[0];
#pragma unroll
  for (int w = 1; w < kStreamWarps; ++w) M = fmaxf(M, sh.red[w]);
  __syncthreads();
  const float ML = M * kLog2e;
  float z = 0.f;
  for (int q = tid; q < npart; q += kStreamThreads) {
    float2 v = __ldcg(&ms[q]);
    if (v.y != 0.f || isnan(v.y)) z += v.y * ex2(fmaf(v.x, kLog2e, -ML));
  }
  z = warp_sum(z);
  if (lane == 0) sh.red[warp] = z;
  // segment starts (seglen is non-zero only at a segment's first chunk; cleared here)
  if (tid == 0) sh.nseg = 0;
  __syncthreads();
  float Z = 0.f;
#pragma unroll
  for (int w = 0; w < kStreamWarps; ++w) Z += sh.red[w];
  for (int c = tid; c < cpr; c += kStreamThreads) {
    int L = __ldcg(&P.seglen[(size_t)row * cpr + c]);
    if (L > 0) {
      int s = atomicAdd(&sh.nseg, 1);
      sh.seg_start[s] = c;
      P.seglen[(size_t)row * cpr + c] = 0;
    }
  }
  __syncthreads();
  const int nlist = sh.nseg * kStreamWarps;

  // (2) exact top-k over the warp lists: warp w merges lists w, w+8, ...
  float lv = -INFINITY;
  int li = kIdxSentinel;
  for (int l = warp; l < nlist; l += kStreamWarps) {
    int c0 = sh.seg_start[l / kStreamWarps];
    size_t base = (((size_t)row * cpr + c0) * kStreamWarps + (l % kStreamWarps)) * k;
    float ev = -INFINITY;
    int ei = kIdxSentinel;
    if (lane < k) {
      ev = __ldcg(&P.segv[base + lane]);
      ei = __ldcg(&P.segi[base + lane]);
    }
    float tv = __shfl_sync(kFull, lv, k - 1);
    int ti = __shfl_sync(kFull, li, k - 1);
    unsigned bal = __ballot_sync(kFull, lane < k && better(ev, ei, tv, ti));
    while (bal) {
      int e = __ffs(bal) - 1;
      bal &= bal - 1;
      float nv = __shfl_sync(kFull, ev, e);
      int ni = __shfl_sync(kFull, ei, e);
      if (!better(nv, ni, tv, ti)) break;  // list entries are sorted: the rest is worse
      warp_insert(lv, li, nv, ni, k, lane);
      tv = __shfl_sync(kFull, lv, k - 1);
      ti = __shfl_sync(kFull, li, k - 1);
    }
  }
  if (lane < k) {
    sh.mlv[warp][lane] = lv;
    sh.mli[warp][lane] = li;
  }
  __syncthreads();
  if (warp == 0) {
    float fv = -INFINITY;
    int fi = kIdxSentinel;
    for (int w = 0; w < kStreamWarps; ++w) {
      float ev = lane < k ? sh.mlv[w][lane] : -INFINITY;
      int ei = lane < k ? sh.mli[w][lane] : kIdxSentinel;
      float tv = __shfl_sync(kFull, fv, k - 1);
      int ti = __shfl_sync(kFull, fi, k - 1);
      unsigned bal = __ballot_sync(kFull, lane < k && better(ev, ei, tv, ti));
      while (bal) {
        int e = __ffs(bal) - 1;
        bal &= bal - 1;
        float nv = __shfl_sync(kFull, ev, e);
        int ni = __shfl_sync(kFull, ei, e);
        if (!better(nv, ni, tv, ti)) break;
        warp_insert(fv, fi, nv, ni, k, lane);
        tv = __shfl_sync(kFull, fv, k - 1);
        ti = __shfl_sync(kFull, fi, k - 1);
      }
    }
    // (3) A1 probabilities and A2 path scores
    int2 fe = P.fr[par][row];
    float pc = P.cum[(size_t)fe.x * P.T + fe.y];
    if (lane < k) {
      float pj = ex2(fmaf(fv, kLog2e, -ML)) / Z;  // p = exp(x - M) / Z   (tau = 1, Q10)
      Cand cd;
      cd.tok = fi;
      cd.p = pj;
      cd.cum = pc * pj;                           // Eq.(3)
      cd.parent = fe.y;
      P.cand[((size_t)(layer - 1) * P.cap_rows + row) * k + lane] = cd;
    }
    if (lane == 0) {
      P.cand_rs[(size_t)(layer - 1) * P.cap_rows + row] = make_int2(fe.x, row - P.fr_off[par][fe.x]);
      P.rowstat[row] = make_float2(M, Z);
      if (!(Z >= 1.0f) || isinf(Z) || isnan(M)) atomicOr(P.err, kErrDraftNaN);  // Q23
      P.row_done[row] = 0;
    }
  }
}

template <bool BF16, bool ALIGNED>
__global__ void __launch_bounds__(kStreamThreads, 2)
expand_kernel(Params P, int layer, const char* __restrict__ logits, long long ld_bytes) {
  constexpr int EPT = Traits<BF16>::EPT;
  __shared__ ExpandShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1;
  const int R = *P.fr_total[par];
  if (R == 0) return;
  const int k = P.k, cpr = P.cpr, CE = P.chunk_elems, V = P.V;
  const long long TOT = (long long)R * cpr;
  const long long lo = TOT * blockIdx.x / gridDim.x;
  const long long hi = TOT * (blockIdx.x + 1) / gridDim.x;
  if (lo >= hi) return;
  if (tid < kStreamWarps) sh.wcnt[tid] = 0;
  if (tid == 0) sh.tau = 0ull;
  __syncthreads();

  uint4 cur[kVecPerThread], nxt[kVecPerThread];
  {
    int row = (int)(lo / cpr), c = (int)(lo % cpr);
    load_chunk<BF16, ALIGNED>(row_ptr(P, par, logits, ld_bytes, row), c * CE, V, tid, cur);
  }

  long long q = lo;
  while (q < hi) {
    const int row = (int)(q / cpr);
    const int c0 = (int)(q % cpr);
    const int nch = (int)min((long long)(cpr - c0), hi - q);
    float lv = -INFINITY;
    int li = kIdxSentinel;
    for (int c = c0; c < c0 + nch; ++c) {
      // prefetch the next unit of this CTA's range
      long long qn = q + (c - c0) + 1;
      if (qn < hi) {
        int rn = (int)(qn / cpr), cn = (int)(qn % cpr);
        load_chunk<BF16, ALIGNED>(row_ptr(P, par, logits, ld_bytes, rn), cn * CE, V, tid, nxt);
      }
      float x[EPT];
      unpack<BF16>(cur, x);
      const int cbase = c * CE;

      // ---- softmax partial of this (chunk, warp): fixed shuffle tree (deterministic) ----
      float m = -INFINITY;
#pragma unroll
      for (int n = 0; n < EPT; ++n) m = fmaxf(m, x[n]);
      const float Mw = warp_max(m);
      float s = 0.f;
      if (Mw != -INFINITY) {
        const float ML = Mw * kLog2e;
#pragma unroll
        for (int n = 0; n < EPT; ++n) s += ex2(fmaf(x[n], kLog2e, -ML));
      }
      s = warp_sum(s);
      if (lane == 0) P.ms[((size_t)row * cpr + c) * kStreamWarps + warp] = make_float2(Mw, s);

      // ---- running top-k of this warp ----
      int excl = -1;
      if (c == c0) {
        int mi = kIdxSentinel;
#pragma unroll
        for (int n = 0; n < EPT; ++n)
          if (x[n] == m && mi == kIdxSentinel) mi = elem_index<BF16>(cbase, tid, n);
        float sv = m;
        int si = mi, src = lane;
        warp_bitonic_desc(sv, si, src, lane);
        lv = lane < k ? sv : -INFINITY;
        li = lane < k ? si : kIdxSentinel;
        unsigned made = 0;
        for (int e = 0; e < k; ++e) made |= 1u << __shfl_sync(kFull, src, e);
        if ((made >> lane) & 1u) excl = mi;
      }
      float tv = __shfl_sync(kFull, lv, k - 1);
      int ti = __shfl_sync(kFull, li, k - 1);
      float fv = tv;  // filter threshold = better of own k-th and the CTA hint
      int fi = ti;
      {
        float hv;
        int hi_;
        unsigned long long hk = *(volatile unsigned long long*)&sh.tau;
        if (hk) {
          split_key(hk, hv, hi_);
          if (better(hv, hi_, fv, fi)) {
            fv = hv;
            fi = hi_;
          }
        }
      }
      bool cl = (m >= fv) && (m == m);
      unsigned pushed = 0u;
      unsigned bal = __ballot_sync(kFull, cl);
      while (bal) {
        bool ovf = false;
        if (cl) {
#pragma unroll
          for (int n = 0; n < EPT; ++n) {
            int gi = elem_index<BF16>(cbase, tid, n);
            if (!((pushed >> n) & 1u) && gi != excl && better(x[n], gi, fv, fi)) {
              int slot = atomicAdd(&sh.wcnt[warp], 1);
              if (slot < kWarpBuf) {
                sh.bufv[warp][slot] = x[n];
                sh.bufi[warp][slot] = gi;
                pushed |= 1u << n;
              } else {
                ovf = true;
              }
            }
          }
        }
        __syncwarp();
        const int cnt = min(sh.wcnt[warp], kWarpBuf);
        for (int e = 0; e < cnt; ++e) {
          float nv = sh.bufv[warp][e];
          int ni = sh.bufi[warp][e];
          if (better(nv, ni, tv, ti)) {
            warp_insert(lv, li, nv, ni, k, lane);
            tv = __shfl_sync(kFull, lv, k - 1);
            ti = __shfl_sync(kFull, li, k - 1);
          }
        }
        __syncwarp();
        if (lane == 0) sh.wcnt[warp] = 0;
        __syncwarp();
        if (better(tv, ti, fv, fi)) {
          fv = tv;
          fi = ti;
        }
        cl = ovf;
        bal = __ballot_sync(kFull, cl);
      }
      if (tv != -INFINITY && lane == 0) atomicMax(&sh.tau, make_key(tv, ti));
#pragma unroll
      for (int j = 0; j < kVecPerThread; ++j) cur[j] = nxt[j];
    }
    // ---- segment end: publish the warp lists, count arrivals ----
    if (lane < k) {
      size_t base = (((size_t)row * cpr + c0) * kStreamWarps + warp) * k;
      P.segv[base + lane] = lv;
      P.segi[base + lane] = li;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      P.seglen[(size_t)row * cpr + c0] = nch;
      __threadfence();
      int old = atomicAdd(&P.row_done[row], nch);
      sh.last = (old + nch == cpr);
      sh.tau = 0ull;
    }
    __syncthreads();
    if (sh.last) {
      __threadfence();
      merge_row(P, layer, par, row, sh);
      __syncthreads();
    }
    q += nch;
  }
}

}  // namespace

int expand_occupancy() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, expand_kernel<true, true>, kStreamThreads, 0);
  return n > 0 ? n : 1;
}

void launch_expand(const Params& P, int layer, const void* logits, long long ld_bytes, bool aligned,
                   int grid, cudaStream_t s) {
  const char* base = static_cast<const char*>(logits);
  if (P.dtype == SMART_BF16) {
    if (aligned) expand_kernel<true, true><<<grid, kStreamThreads, 0, s>>>(P, layer, base, ld_bytes);
    else expand_kernel<true, false><<<grid, kStreamThreads, 0, s>>>(P, layer, base, ld_bytes);
  } else {
    if (aligned) expand_kernel<false, true><<<grid, kStreamThreads, 0, s>>>(P, layer, base, ld_bytes);
    else expand_kernel<false, false><<<grid, kStreamThreads, 0, s>>>(P, layer, base, ld_bytes);
  }
}

}  // namespace smart
