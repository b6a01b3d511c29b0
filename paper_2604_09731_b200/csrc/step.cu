// step.cu — the persistent whole-step kernel behind smart_run_step: one launch runs a whole decode
// step of the SMART controller (Algorithm 1) for a batch — d layers of A1+A2 (top-k +
// softmax of every frontier row; cum = cum(parent) * p, Eq.(3)) and A3-A6
// (select_core.cuh), then A7 (mask, position ids, parents) and A8 (the greedy
// longest-accepted-path walk on the target logits, P:453 / S:383).
//
// Layout: gridDim.x - 1 streaming CTAs and one selection CTA, all co-resident
// (grid = SMs x occupancy).  Layers are separated by flags in global memory, not by kernel
// boundaries, and every cross-SM hop is a self-validating tagged word or 16-byte line (tag =
// launch epoch and layer) polled with relaxed loads: no arrival counters, no fences per layer.
//  * streaming CTA s, layer l with R frontier rows: team size t = min(cpr, S / R, 32) (t = 1 when
//    R > S); CTA s is member s % t of team s / t, which streams rows team, team + S/t, ...; the
//    member's slice of a row is chunks [m cpr / t, (m+1) cpr / t).  A producer lane bulk-copies the
//    chunks into the TMA ring (cp.async.bulk + mbarrier), 8 consumer warps reduce them
//    (expand_core.cuh) and write the slice's top-k list and per-chunk softmax partials as tagged
//    lines.  Member 0 of the team then polls the row's t lists and cpr partials, merges them (one
//    warp: Z and a k-round tournament) and writes the row's k candidates (token, p) as tagged
//    lines.  Layer 1's rows are the roots (r, 0); for layer l >= 2 the producer lane polls
//    flag[l] and its rows' tagged frontier entries; consumers learn the row count through a
//    shared-memory mbarrier.
//  * the selection CTA keeps the per-request state, polls the layer's R * k candidate lines into
//    its staged records (cum = cum(parent) * p, Eq.(3)), runs A3-A6 (select_layer) and publishes
//    the next frontier as tagged entries and flag[l+1] = (tag << 32 | R').  After the last layer it
//    writes the verify-row table and publishes flag[kVerifySlot]; the streaming CTAs stream every
//    tree row of the target logits (exact argmax, red.max on the row's slot, then one release word
//    per CTA) while it writes the mask outputs; then it walks.
#include <cstdlib>

#include "expand_core.cuh"
#include "select_core.cuh"
#include "verify_core.cuh"

namespace smart {

namespace {

constexpr int kStepThreads = kLayerThreads;  // 8 consumer warps + 1 producer warp
constexpr int kProducerWarp = kConsumerWarps;
constexpr int kTeamMax = 32;                  // slices per row (one list per lane in the merge)

struct __align__(16) StepShared {
  ConsShared cs;
  float2 msl[kMaxCpr * kConsumerWarps];  // (chunk, warp) softmax partials of the current slice
  // producer -> consumers: the value of event e (the row count of layer e + 2, or the verify rows)
  // is rv[e], published by one arrive on its own mbarrier evb[e] (each completes exactly once per
  // launch, so there is no phase aliasing however far ahead the producer runs)
  int rv[SMART_MAX_DEPTH + 2];
  uint64_t evb[SMART_MAX_DEPTH + 2];
};
// the team merge (member 0 of a row's team) stages the row's t slice lists (stride kp) and cpr
// partials in the warps' top-k buffers (dead between slices): no extra shared memory, so two
// streaming CTAs still fit one SM
static_assert(sizeof(WarpTopk) * kConsumerWarps >= (size_t)kTeamMax * kMaxK * 8 + kMaxCpr * sizeof(float2),
              "team-merge staging must fit the warp buffers");
__device__ __forceinline__ unsigned long long* merge_keys(StepShared& sh) {
  return reinterpret_cast<unsigned long long*>(&sh.cs.w[0]);
}
__device__ __forceinline__ float2* merge_ms(StepShared& sh) {
  return reinterpret_cast<float2*>(reinterpret_cast<char*>(&sh.cs.w[0]) + (size_t)kTeamMax * kMaxK * 8);
}

__device__ __forceinline__ void post_event(StepShared& sh, int e, int v) {
  sh.rv[e] = v;
  mbar_arrive(&sh.evb[e]);  // release (CTA scope)
}
__device__ __forceinline__ int wait_event(StepShared& sh, int e) {
  mbar_wait(&sh.evb[e], 0u);  // acquire (CTA scope)
  return sh.rv[e];
}

__host__ __device__ inline int team_size(int R, int S, int cpr) {
  if (R <= 0 || R >= S) return 1;
  int t = S / R;
  if (t > cpr) t = cpr;
  if (t > kTeamMax) t = kTeamMax;
  return t;
}

// balanced contiguous unit ranges over g = min(gmax, ceil(total / min_units)) CTAs
__host__ __device__ inline int range_ctas(int total, int gmax, int min_units) {
  const int g = (total + min_units - 1) / min_units;
  return g < gmax ? g : gmax;
}
__device__ __forceinline__ RowRange range_of(int total, int gmax, int min_units, int b) {
  const int g = range_ctas(total, gmax, min_units);
  RowRange r;
  if (b >= g) {
    r.lo = r.hi = 0;
    return r;
  }
  const int base = total / g, rem = total - base * g;
  r.lo = b * base + min(b, rem);
  r.hi = r.lo + base + (b < rem ? 1 : 0);
  return r;
}

// Polls use relaxed loads and one acquire fence once the value is seen (relaxed load + fence =
// acquire pattern): an ld.acquire per poll compiles to LDG + CCTL.IVALL, and a stream of L1
// invalidations from a spinning lane slows every warp sharing the SM.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Polls are bounded (~2^24 tries, seconds): a broken protocol sets the sticky kErrTimeout
// flag (SMART_EDEVICE from smart_get_stats) and lets the step run out instead of hanging the GPU.
constexpr unsigned kPollLimit = 1u << 24;

// poll a (tag << 32 | value) flag of this launch; returns the value (0 on timeout).  No acquire
// fence: after a flag only self-validating words are read
__device__ __forceinline__ int wait_tag_relaxed(const unsigned long long* f, unsigned tag, int* err) {
  for (unsigned it = 0;; ++it) {
    const unsigned long long v = ld_relaxed_u64(f);
    if ((unsigned)(v >> 32) == tag) return (int)(unsigned)v;
    if (it > kPollLimit) {
      atomicOr(err, kErrTimeout);
      return 0;
    }
    __nanosleep(20);
  }
}
// a frontier entry's tag: unique per (launch, layer)
__device__ __forceinline__ unsigned entry_tag(unsigned tag, int layer) { return (tag << 5) | (unsigned)layer; }
// poll a tagged frontier entry; returns (r << 10 | node)
__device__ __forceinline__ unsigned wait_entry(const unsigned long long* e, unsigned etag, int* err) {
  for (unsigned it = 0;; ++it) {
    const unsigned long long v = ld_relaxed_u64(e);
    if ((unsigned)(v >> 32) == etag) return (unsigned)v;
    if (it > kPollLimit) {
      atomicOr(err, kErrTimeout);
      return 0u;
    }
  }
}

// Self-validating 16-byte lines {a, tag, b, tag}: each 8-byte half carries the tag, so a torn
// access is caught.  The slice lists / partials and the merged candidates of a layer are polled on
// the data itself: no arrival counter (serialised at one L2 address) and no release/acquire fence
// on the hop (tools/ubench/handoff.cu: 16 slices, 1.47 us with counter + fences, 0.1 us tagged).
__device__ __forceinline__ void st_line(uint4* p, unsigned a, unsigned b, unsigned tag) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(tag), "r"(b), "r"(tag)
               : "memory");
}
__device__ __forceinline__ uint2 wait_line(const uint4* p, unsigned tag, int* err) {
  for (unsigned it = 0;; ++it) {
    unsigned a, t0, b, t1;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(t0), "=r"(b), "=r"(t1)
                 : "l"(p)
                 : "memory");
    if (t0 == tag && t1 == tag) return make_uint2(a, b);
    if (it > kPollLimit) {
      atomicOr(err, kErrTimeout);
      return make_uint2(0u, 0u);
    }
    __nanosleep(32);  // a waiting warp must not take issue slots from the SM's streaming warps
  }
}

// the step kernel's frontier publication: every entry also as a self-validating tagged word, the
// row count as a tagged flag, all with plain stores (no release fence on the critical path: what
// the streaming CTAs read behind the flag is the tagged entries themselves)
struct StepPub {
  const Params* P;
  unsigned tag;
  int layer;
  __device__ void entry(int pos, int r, int node) const {
    if (layer < P->d)
      st_relaxed_u64(&P->fr_tag[pos],
                     ((unsigned long long)entry_tag(tag, layer + 1) << 32) | ((unsigned)r << 10) | (unsigned)node);
  }
  __device__ void operator()(int tot) const {
    if (layer < P->d) st_relaxed_u64(&P->ctl->flag[layer + 1], ((unsigned long long)tag << 32) | (unsigned)tot);
  }
};


// timeline probes (SMART_PROBES=1 builds only): dbg[256 + 16 * layer + slot], globaltimer ns;
// "max" slots keep the latest time, "min" slots the complement of the earliest (atomicMax of ~t)
enum { kPbArrived = 0, kPbMerged = 1, kPbPublished = 2, kPbFlagMin = 3, kPbFlagMax = 4, kPbSliceMax = 5,
       kPbChunkMin = 6, kPbChunkMax = 7, kPbSelDone = 8, kPbSync1 = 9, kPbStaged = 10, kPbConsumed1 = 11,
       kPbPosted = 12, kPbTeamIn = 13, kPbTeamOut = 14 };
__device__ __forceinline__ unsigned smid_reg() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void pb_max(const Params& P, int layer, int slot) {
  if (SMART_PROBES && P.dbg) atomicMax(&P.dbg[256 + 16 * layer + slot], gtime());
}
__device__ __forceinline__ void pb_min(const Params& P, int layer, int slot) {
  if (SMART_PROBES && P.dbg) atomicMax(&P.dbg[256 + 16 * layer + slot], ~gtime());
}

// ---------------------------------------------------------------------------------------------
// team merge (A1 finish + A2 of one row), by member 0 of the row's team once its own slice is
// out: the row's t slice lists and cpr per-chunk partials are polled as tagged lines into shared
// memory, warp 0 merges them (k-round tournament, expand_core.cuh) and writes the row's k
// candidates (token, p) as tagged lines; the selection CTA forms cum = cum(parent) * p (Eq.(3))
// from its own frontier.  Rows merge in parallel on their teams instead of one after another on
// the selection CTA.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void team_merge(const Params& P, StepShared& sh, int row, int t, unsigned lt, int layer) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const int k = P.k, kp = list_stride(k), cpr = P.cpr;
  const int nkl = t * k, nl = nkl + cpr;
  const uint4* gk = P.seg_key + (size_t)row * t * k;
  const uint4* gm = P.seg_ms + (size_t)row * cpr;
  unsigned long long* mk = merge_keys(sh);
  float2* mm = merge_ms(sh);
  for (int e = tid; e < nl; e += kConsumers) {
    if (e < nkl) {
      const uint2 v = wait_line(gk + e, lt, P.err);
      mk[(e / k) * kp + e % k] = ((unsigned long long)v.y << 32) | v.x;
    } else {
      const uint2 v = wait_line(gm + (e - nkl), lt, P.err);
      mm[e - nkl] = make_float2(__uint_as_float(v.x), __uint_as_float(v.y));
    }
  }
  consumer_sync();
  if (tid == 0) pb_max(P, layer, kPbTeamIn);  // all lists in (latest row)
  if (warp == 0) {
    uint4* gc = P.seg_cand + (size_t)row * k;
    const bool ok = merge_row_tournament(
        k, cpr, t, 1.f,
        [&](int c) {
          const float2 v = mm[c];
          return make_float4(v.x, v.y, 0.f, 0.f);
        },
        mk, [&](int rank, int tok, float p, float) { st_line(gc + rank, (unsigned)tok, __float_as_uint(p), lt); });
    if (!ok && (tid & 31) == 0) atomicOr(P.err, kErrDraftNaN);  // Q23
  }
  consumer_sync();  // the warp buffers are the next slice's again
  if (tid == 0) pb_max(P, layer, kPbTeamOut);  // row candidates out (latest row)
}

// ---------------------------------------------------------------------------------------------
// streaming CTA
// ---------------------------------------------------------------------------------------------
template <bool BF16>
__device__ void stream_role(const Params& P, char* dsm, const char* __restrict__ draft, long long ld_d,
                            const char* __restrict__ target, long long ld_t, unsigned tag) {
  char* ring = dsm;
  StreamPipe& pipe = *reinterpret_cast<StreamPipe*>(dsm + kStages * kChunkBytes);
  StepShared& sh = *reinterpret_cast<StepShared*>(dsm + kStages * kChunkBytes + sizeof(StreamPipe));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = P.step_S, s = (int)blockIdx.x;
  const int k = P.k, cpr = P.cpr, kp = list_stride(k), T = P.T;
  const long long row_bytes = (long long)P.V * (BF16 ? 2 : 4);
  int R = P.d > 0 ? P.b_loc : 0;
  int layer = 1;

  if (warp == kProducerWarp) {
    if (lane != 0) return;
    int i = 0;  // the CTA's running chunk counter (ring stage and phase), same sequence as the consumers
    int ev = 0;
    auto issue = [&](const char* base, int c) {
      const int st = i % kStages;
      mbar_wait(&pipe.empty[st], ((uint32_t)(i / kStages) & 1u) ^ 1u);
      const long long off = (long long)c * kChunkBytes;
      const uint32_t bytes = (uint32_t)min((long long)kChunkBytes, row_bytes - off);
      mbar_expect_tx(&pipe.full[st], bytes);
      bulk_g2s(ring + (size_t)st * kChunkBytes, base + off, bytes, &pipe.full[st]);
      ++i;
    };
    while (R > 0 && layer <= P.d) {
      const int t = team_size(R, S, cpr);
      const int nteams = S / t, team = s / t, member = s - team * t;
      const int mlo = member * cpr / t, mhi = (member + 1) * cpr / t;
      if (team < nteams) {
        for (int row = team; row < R; row += nteams) {
          int r = row, node = 0;  // layer 1: the roots
          if (layer > 1) {  // the row's self-validating frontier entry
            const unsigned w = wait_entry(&P.fr_tag[row], entry_tag(tag, layer), P.err);
            r = (int)(w >> 10);
            node = (int)(w & 1023u);
          }
          const char* base = P.row_mode == SMART_ROWS_POSITION ? draft + ((long long)r * P.d + (layer - 1)) * ld_d
                                                                : draft + ((long long)r * T + node) * ld_d;
          for (int c = mlo; c < mhi; ++c) issue(base, c);
        }
      }
      const int Rn = layer < P.d ? wait_tag_relaxed(&P.ctl->flag[layer + 1], tag, P.err) : 0;
      if (layer < P.d) {
        pb_min(P, layer + 1, kPbFlagMin);
        pb_max(P, layer + 1, kPbFlagMax);
      }
      post_event(sh, ev++, Rn);
      R = Rn;
      ++layer;
    }
    const int NR = wait_tag_relaxed(&P.ctl->flag[kVerifySlot], tag, P.err);
    pb_min(P, kVerifySlot, kPbFlagMin);
    pb_max(P, kVerifySlot, kPbFlagMax);
    post_event(sh, ev++, NR);
    if (NR > 0) {
      const RowRange rr = range_of(NR * cpr, S, P.min_units, s);
      int row = rr.lo / cpr, c = rr.lo - row * cpr;
      const char* base = nullptr;
      for (int q = rr.lo; q < rr.hi; ++q) {
        if (q == rr.lo || c == 0) {  // the row's self-validating verify entry
          const unsigned w = wait_entry(&P.fr_tag[row], entry_tag(tag, 31), P.err);
          base = target + ((long long)(w >> 10) * T + (w & 1023u)) * ld_t;
        }
        issue(base, c);
        if (++c == cpr) {
          c = 0;
          ++row;
        }
      }
    }
    return;
  }

  // ---- consumer warps ----
  int i = 0, ev = 0, wcnt = 0;
  float wrun = -INFINITY;  // the warp's running max over the current slice
  while (R > 0 && layer <= P.d) {
    const int t = team_size(R, S, cpr);
    const int nteams = S / t, team = s / t, member = s - team * t;
    const int mlo = member * cpr / t, mhi = (member + 1) * cpr / t;
    if (team < nteams) {
      for (int row = team; row < R; row += nteams) {
        unsigned long long bound = 0ull;  // lower bound of the slice's k-th best key
        for (int c = mlo; c < mhi; ++c, ++i) {
          const int st = i % kStages;
          const char* stage = ring + (size_t)st * kChunkBytes;
          mbar_wait(&pipe.full[st], ((uint32_t)(i / kStages)) & 1u);
          if (tid == 0 && c == mlo) {
            pb_min(P, layer, kPbChunkMin);
            pb_max(P, layer, kPbChunkMax);
            if (SMART_PROBES && P.dbg && layer == 2 && P.debug_mode != 9) P.dbg[1024 + 4 * s] = gtime();
          }
          uint4 raw[kVecPerThread];
          const uint4* sv = reinterpret_cast<const uint4*>(stage);
#pragma unroll
          for (int j = 0; j < kVecPerThread; ++j) raw[j] = sv[j * kConsumers + tid];
          consume_chunk<BF16, true>(P, sh.cs, sh.msl, raw, stage, nullptr, c, mlo, mhi, i, wcnt, bound, wrun);
          __syncwarp();
          if (tid == 0 && c == mlo) pb_max(P, layer, kPbConsumed1);
          if (SMART_PROBES && P.dbg && layer == 2 && P.debug_mode != 9 && tid == 0 && c == mlo) P.dbg[1024 + 4 * s + 1] = gtime();
          if (lane == 0) mbar_arrive(&pipe.empty[st]);  // release the stage
        }
        // slice end: the CTA's top-k and per-chunk partials straight to global memory
        slice_end_post(sh.cs, k, wcnt);
        if (tid == 0) pb_max(P, layer, kPbPosted);
        if (SMART_PROBES && P.dbg && layer == 2 && P.debug_mode != 9 && tid == 0) {
          P.dbg[1024 + 4 * s + 2] = gtime();
          P.dbg[1024 + 4 * s + 3] = (unsigned long long)(mhi - mlo) | ((unsigned long long)row << 8) | ((unsigned long long)smid_reg() << 16);
        }
        const unsigned lt = entry_tag(tag, layer);
        uint4* gk = P.seg_key + (size_t)(row * t + member) * k;
        uint4* gm = P.seg_ms + (size_t)row * cpr + mlo;
        slice_end_merge(
            sh.cs, sh.msl, k, mhi - mlo,
            [&](int rank, unsigned long long key) {
              if (rank < k) st_line(gk + rank, (unsigned)key, (unsigned)(key >> 32), lt);
            },
            [&](int cc, float Mc, float Sc) { st_line(gm + cc, __float_as_uint(Mc), __float_as_uint(Sc), lt); });
        consumer_sync();  // sh.cl / msl are reused by the next slice
        if (tid == 0) {
          pb_max(P, layer, kPbSliceMax);
          sh.cs.tau = 0ull;  // next slice (read only after the next slice's first barrier)
        }
        if (member == 0) team_merge(P, sh, row, t, lt, layer);
      }
    }
    R = wait_event(sh, ev++);
    ++layer;
  }
  // ---- A8 stream: every tree row of the target logits, exact argmax per row segment ----
  // The loop's first pass is dry: one chunk of stale stage data through the same code, results
  // dropped, while the selection finishes the trees -- the first real chunk then runs from a warm
  // instruction cache (cold, it took 1.4 us against 0.45 us for the later chunks).
  bool dry = true;
  RowRange rr;
  rr.lo = 0;
  rr.hi = 1;
  int nanf = 0;
  int q = 0, row = 0, c0 = 0;
  bool vpb = false;
  for (;;) {
    if (q >= rr.hi) {
      if (!dry) break;
      dry = false;
      nanf = 0;
      const int NR = wait_event(sh, ev++);
      if (NR <= 0) return;
      rr = range_of(NR * cpr, S, P.min_units, s);
      if (rr.lo >= rr.hi) return;
      q = rr.lo;
      row = rr.lo / cpr;
      c0 = rr.lo - row * cpr;
      vpb = SMART_PROBES && P.dbg && P.debug_mode == 9 && tid == 0;  // per-CTA A8 probes
      if (vpb) P.dbg[1024 + 4 * s + 3] = (unsigned long long)(rr.hi - rr.lo) | ((unsigned long long)row << 8) |
                                         ((unsigned long long)smid_reg() << 16);
    }
    const int nch = dry ? 1 : min(cpr - c0, rr.hi - q);
    int2 rn = make_int2(0, 0);
    if (!dry) {
      const unsigned rw = wait_entry(&P.fr_tag[row], entry_tag(tag, 31), P.err);
      rn = make_int2((int)(rw >> 10), (int)(rw & 1023u));
    }
    float bv = -INFINITY;
    int bi = kIdxSentinel;
    for (int c = c0; c < c0 + nch; ++c) {
      const int st = i % kStages;
      if (!dry) mbar_wait(&pipe.full[st], ((uint32_t)(i / kStages)) & 1u);
      uint4 raw[kVecPerThread];
      const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)st * kChunkBytes);
#pragma unroll
      for (int j = 0; j < kVecPerThread; ++j) raw[j] = sv[j * kConsumers + tid];
      __syncwarp();
      if (!dry && lane == 0) mbar_arrive(&pipe.empty[st]);
      if (vpb && q == rr.lo && c == c0) P.dbg[1024 + 4 * s] = gtime();  // first chunk landed
      verify_chunk<BF16, false>(raw, c * P.chunk_elems, P.V, tid, 0u, 1.f, bv, bi, nanf);
      if (vpb && q == rr.lo && c == c0) P.dbg[1024 + 4 * s + 1] = gtime();  // and consumed
      if (!dry) ++i;
    }
    if (!dry && lane == 0 && bi != kIdxSentinel) {
      const unsigned long long key = ((unsigned long long)vkey_orderable(bv) << 32) | (0xffffffffu - (unsigned)bi);
      asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(P.vbest + (size_t)rn.x * T + rn.y), "l"(key)
                   : "memory");
    }
    q += nch;
    ++row;
    c0 = 0;
  }
  if (nanf) atomicOr(P.err, kErrTargetNaN);
  if (vpb) P.dbg[1024 + 4 * s + 2] = gtime();  // last chunk consumed
  consumer_sync();
  if (tid == 0) {
    pb_max(P, kVerifySlot, kPbSliceMax);
    // release (cumulative over the barrier: the CTA's red.max on the row slots), one word per CTA
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&P.ctl->vdone[s]), "l"((unsigned long long)tag << 32)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------------------------
// selection CTA
// ---------------------------------------------------------------------------------------------

struct MergeLayout {
  int2* fe;    // [rows] frontier entry (request, node)
  float* pc;   // [rows] parent cum
  int* slot;   // [rows] frontier slot within the request
};

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t merge_bytes(int rows_cap) {
  return a16((size_t)rows_cap * 8) + a16((size_t)rows_cap * 4) + a16((size_t)rows_cap * 4);
}

__device__ inline MergeLayout merge_layout(char* p, int rows_cap) {
  MergeLayout M;
  M.fe = reinterpret_cast<int2*>(p);
  p += a16((size_t)rows_cap * 8);
  M.pc = reinterpret_cast<float*>(p);
  p += a16((size_t)rows_cap * 4);
  M.slot = reinterpret_cast<int*>(p);
  return M;
}

// ---------------------------------------------------------------------------------------------
// select_small: A3-A6 of one layer for small batches (one rank, <= 32 requests, NODE_SUM, PREFIX
// or FROZEN) -- the same decisions, node numbering, fp64 associations and trace as select_layer,
// computed on the few candidates that can matter, in one warp, with the per-request state in
// registers (lane r of warp 0 holds request r).  Every dependent warp collective costs ~30-50
// cycles and every block barrier ~40 (profiles/r02c_ubench_latency.txt), so this path is a few
// warp-wide steps instead of select_layer's barrier-separated block phases.
//  * theta (known before the layer's candidates arrive): Eq.(16) admits the candidate at sorted
//    position j only if alpha c_T b_j C(N0+j) > (rhs0 + c_T before_j) dc(N0+j) with before_j >= 0,
//    so every admitted candidate has b > theta = min_j rhs0 dc(N0+j) / (alpha c_T C(N0+j))
//    (FROZEN: the j = 0 term is its whole rule).  Every candidate that beats an above-theta one
//    within its request (A3) or globally (A4) is itself above theta, so ranks, eligibility and the
//    order of the above-theta eligible candidates are exact among them alone, and the first sorted
//    position at or below theta fails the rule: the cut lies in the above-theta prefix (cfg3: 30
//    above-theta candidates of 256 at layer 1, 28 admitted).
//  * one warp, lane = one above-theta candidate: "better than" / same-request / lower-index masks,
//    within-request rank = popc(better & same) < e_r (A3, Eq.(8)), sorted position = popc(better &
//    eligible) (A4), tile 0 of the block path's A5 scan and rule (same association), node index =
//    admitted candidates of the request with a lower canonical index (A6).
//  * trace argmax_j S_j: exact over the above-theta prefix; beyond it every benefit is <= theta, so
//    S_j <= c_T (omega b + E0 + P + (j - n) theta) / C(N0+j); if that bound stays below the best S
//    (1e-9 margin) the argmax is final, else the full list is rebuilt (small_trace_full).
// Falls back (returns false; the records are staged for select_layer) when theta is not usable,
// more than 32 candidates are above it, or the eligible list is longer than kA5Par.
// ---------------------------------------------------------------------------------------------
struct SmallState {  // lane r of warp 0: request r's state before the layer
  int cnt, off, nd, fin;
  double E;
};
struct SmallShared {
  double theta, E0, th_cut, th_arg;
  long long N0, N0next;
  int ne, n_above, need_full, bestj;
  int a[32];
  int vpub;    // the verify rows are published (select_small, after the last layer)
  int nn[32];  // node counts after the last layer (lane r of warp 0), for the verify-row table
  __align__(16) unsigned long long akeys[64];
};

__device__ __forceinline__ void small_state_load(const Params& P, int par, int lane, SmallState& st) {
  if (lane < P.b_loc) {
    st.cnt = P.fr_cnt[par][lane];
    st.off = P.fr_off[par][lane];
    st.nd = P.n_nodes[lane] - 1;
    st.fin = P.finished[lane];
    st.E = P.E_r[lane];
  } else {
    st.cnt = st.off = st.nd = st.fin = 0;
    st.E = 0.0;
  }
}

// the full sorted eligible list of a layer for the trace argmax (rare: only when the bound of
// select_small cannot exclude the positions below theta); all 256 threads, block-path association
__device__ __forceinline__ void small_trace_full(const Params& P, char* dsm, SmallShared& sh, int nct, int ne, double E0,
                                              int bc) {
  SelLayout L = sel_layout(dsm, P.b_loc, P.cap_rows * P.k, P.k, P.sort_cap);
  L.keys = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(L.E) + sel_align((size_t)P.b_loc * 8));
  L.keys2 = L.keys + P.sort_cap;
  const int* ebase = L.base;
  __shared__ double tile[kA5Par / 32], wS[kConsumerWarps];
  __shared__ int wJ[kConsumerWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, k = P.k, bl = P.b_loc;
  for (int q = tid; q < nct; q += kConsumers) {
    const int r = L.rreq[q / k];
    const int s0 = L.off[r] * k, s1 = s0 + L.cnt[r] * k;
    const int e_r = (r + 1 < bl ? ebase[r + 1] : ne) - ebase[r];
    const float b = L.cb[q];
    int rank = 0;
    for (int j = s0; j < s1; ++j) {
      const float bj = L.cb[j];
      rank += (bj > b) || (bj == b && j < q);
    }
    if (rank < e_r) L.keys2[ebase[r] + rank] = sel_key(b, P.b_off + r, q - s0);
  }
  consumer_sync();
  for (int i = tid; i < ne; i += kConsumers) {
    const unsigned long long key = L.keys2[i];
    int rank = 0;
    for (int f = 0; f < ne; ++f) rank += L.keys2[f] < key;
    L.keys[rank] = key;
  }
  consumer_sync();
  const bool act = tid < ne;
  const double bj = act ? (double)sel_key_b(L.keys[tid]) : 0.0;
  double incl = bj;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += u;
  }
  double excl = __shfl_up_sync(kFull, incl, 1);
  if (lane == 0) excl = 0.0;
  if (lane == 31) tile[warp] = incl;
  consumer_sync();
  double before = 0.0;
  for (int w = 0; w < warp; ++w) before += tile[w];
  before += excl;
  double bestS = -1.0;
  int bestj = 1 << 30;
  if (act) {
    const double C = L.ctab[tid + 1];
    bestS = C > 0.0 ? P.c_T * ((double)P.omega * bc + (E0 + before + bj)) / C : 0.0;
    bestj = tid + 1;
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
    wS[warp] = bestS;  // per-warp winners
    wJ[warp] = bestj;
  }
  consumer_sync();
  if (tid == 0) {
    const double C0 = L.ctab[0];
    double S = C0 > 0.0 ? P.c_T * ((double)P.omega * bc + E0) / C0 : 0.0;
    int j = 0;
    for (int w = 0; w < kConsumerWarps; ++w)
      if (wJ[w] <= ne && (wS[w] > S || (wS[w] == S && wJ[w] < j))) {
        S = wS[w];
        j = wJ[w];
      }
    sh.bestj = j;
  }
  consumer_sync();
}

template <class Pub>
__device__ __forceinline__ bool select_small(const Params& P, int layer, int R, char* dsm, const MergeLayout& M,
                                             const MergeLayout& Mn, bool rows_in_smem, SmallState& st,
                                             SmallShared& sh, unsigned tag, Pub pub, bool verify) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (layer - 1) & 1, npar = layer & 1;
  const int k = P.k, bl = P.b_loc, nct = R * k, T = P.T;
  const size_t lbase = (size_t)(layer - 1) * P.cap_rows * k;
  SelLayout L = sel_layout(dsm, bl, P.cap_rows * k, k, P.sort_cap);
  L.keys = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(L.E) + sel_align((size_t)bl * 8));
  L.keys2 = L.keys + P.sort_cap;
  int4* const crec = reinterpret_cast<int4*>(L.keys + 2 * (size_t)P.sort_cap);
  const int bc = (P.cost_scope == SMART_COST_LOCAL) ? bl : P.b_glob;
  const double ac = P.alpha * P.c_T;
  // the frontier buffers of this layer (par) and the next (npar), selected without indexing the
  // kernel parameter arrays by a runtime value (that copies them to local memory)
  int2* const fr_p = par ? P.fr[1] : P.fr[0];
  float* const frc_p = par ? P.fr_cum[1] : P.fr_cum[0];
  int* const fro_p = par ? P.fr_off[1] : P.fr_off[0];
  int2* const fr_n = npar ? P.fr[1] : P.fr[0];
  float* const frc_n = npar ? P.fr_cum[1] : P.fr_cum[0];
  int* const fro_n = npar ? P.fr_off[1] : P.fr_off[0];
  int* const frn_n = npar ? P.fr_cnt[1] : P.fr_cnt[0];
  int* const frt_n = npar ? P.fr_total[1] : P.fr_total[0];
  stamp(P, tid == 0, 9);
  // ---- before the candidates: the cost window from N0 (all threads, one round of loads); A3
  // budgets (lane r), E0, theta and the argmax threshold (warp 0); the rows' descriptors ----
  {
    const long long N0w = sh.N0next;  // drafted nodes before the layer (the last layer's N0 + js)
    const int ncw = min(nct, P.sort_cap) + 2;
    for (int j = tid; j < ncw; j += kConsumers) {
      const long long N = min(N0w + j, (long long)P.n_cost - 1);
      L.ctab[j] = P.cost_tab[N];
      L.dtab[j] = P.dc_tab[N];
    }
  }
  consumer_sync();
  int e = 0, eb = 0;
  if (warp == 0) {
    if (lane < bl) {
      int q = P.B - st.nd;
      if (q > P.Wq) q = P.Wq;
      if (q < 0) q = 0;
      e = min(q, st.cnt * k);  // e_r = min(B - n_r, W, |U_r|)
    }
    int incl = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += u;
    }
    eb = incl - e;
    const int ne = __shfl_sync(kFull, incl, 31);
    int nd = lane < bl ? st.nd : 0;
    double Ev = lane < bl ? st.E : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      nd += __shfl_xor_sync(kFull, nd, o);
      Ev += __shfl_xor_sync(kFull, Ev, o);  // warp_det_sum of one tile (Q13)
    }
    const long long N0 = nd;
    const double rhs0 = P.c_T * ((double)P.omega * bc + Ev);
    const int ncw = min(nct, P.sort_cap) + 2;
    double th = INFINITY;
    bool ok = ac > 0.0 && P.c_T >= 0.0 && rhs0 >= 0.0;
#pragma unroll 1
    for (int j = lane; j < ncw; j += 32) {
      const double C = L.ctab[j], dcj = L.dtab[j];
      // a float reciprocal (rel. error < 1e-7; the 1e-5 margin below covers it): a
        // correctly rounded fp64 one is a ~30-instruction call per entry
        const double tj = C > 0.0 ? rhs0 * dcj * (double)__frcp_rn((float)(ac * C)) : 0.0;
      ok = ok && dcj >= 0.0 && tj == tj;
      th = fmin(th, tj);
    }
    // argmax threshold: on a convex window (dC nondecreasing over prefix lengths 0..ne+1) with
    // sorted benefits, S_j is unimodal (S_{j+1} lies between S_j and b_j / dC_j), and a step can
    // raise S only if b_j > s_j dC_j >= s_0 min dC (s = S / c_T): every benefit <= th2 = s_0 min dC
    // ends the rise for good; 1e-6 below keeps the computed S of later prefixes under the maximum
    // (the convexity test allows 1e-9 of rounding in dC: exactly linear costs qualify)
    bool cvx = L.ctab[0] > 0.0;
    double dmin = INFINITY;
#pragma unroll 1
    for (int j = lane; j <= ne; j += 32) {
      const double d0 = L.ctab[j + 1] - L.ctab[j];
      dmin = fmin(dmin, d0);
      if (j + 1 <= ne) cvx = cvx && (L.ctab[j + 2] - L.ctab[j + 1]) >= d0 - 1e-9 * fabs(d0);  // convex up to rounding
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      th = fmin(th, __shfl_xor_sync(kFull, th, o));
      dmin = fmin(dmin, __shfl_xor_sync(kFull, dmin, o));
    }
    ok = __all_sync(kFull, ok) && th > 0.0 && th < INFINITY;
    cvx = __all_sync(kFull, cvx) && dmin > 0.0 && dmin < INFINITY;
    if (lane == 0) {
      const double thc = ok ? th * (1.0 - 1e-5) : -1.0;
      const double th2 = cvx ? ((double)P.omega * bc + Ev) / L.ctab[0] * dmin * (1.0 - 1e-6) : -1.0;
      sh.th_cut = thc;
      sh.th_arg = th2;
      sh.theta = (thc >= 0.0 && th2 > 0.0) ? fmin(thc, th2) : thc;  // the screening threshold
      sh.E0 = Ev;
      sh.N0 = N0;
      sh.ne = ne;
      sh.n_above = 0;
    }
  }
  if (!rows_in_smem) {  // after a block-path layer: the rows from its global frontier
    for (int row = tid; row < R; row += kConsumers) {
      const int2 fe = fr_p[row];
      M.fe[row] = fe;
      M.pc[row] = frc_p[row];
      M.slot[row] = row - fro_p[fe.x];
    }
  }
  consumer_sync();
  stamp(P, tid == 0, 10);
  if (tid == 0) pb_max(P, layer, kPbSync1);
  // ---- the rows' merged candidates: records, benefits, screened keys (warp ballots) ----
  const double theta = sh.theta;
  {
    const unsigned lt = entry_tag(tag, layer);
#pragma unroll 1
    for (int q0 = warp * 32; q0 < nct; q0 += kConsumers) {
      const int q = q0 + lane;
      bool ab = false;
      unsigned long long key = 0ull;
      if (q < nct) {
        const uint2 v = wait_line(P.seg_cand + q, lt, P.err);
        const int row = q / k, h = q - row * k;
        const int2 fe = M.fe[row];
        const float cum = __fmul_rn(M.pc[row], __uint_as_float(v.y));  // Eq.(3)
        crec[q] = make_int4((int)v.x, (int)v.y, __float_as_int(cum), fe.y);
        L.cb[q] = cum;  // NODE_SUM: b = cum (Eq.(13) with D = 1)
        if (h == 0) L.rreq[row] = fe.x;
        P.cand_adm[lbase + q] = 0;
        ab = (double)cum > theta;
        key = sel_key(cum, P.b_off + fe.x, M.slot[row] * k + h);
      }
      const unsigned m = __ballot_sync(kFull, ab);
      if (m) {
        int pos = 0;
        if (lane == __ffs(m) - 1) pos = atomicAdd(&sh.n_above, __popc(m));
        pos = __shfl_sync(kFull, pos, __ffs(m) - 1) + __popc(m & ((1u << lane) - 1u));
        if (ab && pos < 64) sh.akeys[pos] = key;
      }
    }
  }
  consumer_sync();
  stamp(P, tid == 0, 11);
  if (tid == 0) pb_max(P, layer, kPbMerged);
  const int nA = sh.n_above, ne = sh.ne;
  if (theta < 0.0 || nA > 32 || ne > kA5Par) return false;

  if (warp == 0) {
    const double E0 = sh.E0, th_cut = sh.th_cut, th_arg = sh.th_arg;
    const long long N0 = sh.N0;
    const double rhs0 = P.c_T * ((double)P.omega * bc + E0);
    // ---- A3 + A4 among the screened candidates (lane = one of them) ----
    const bool own = lane < nA;
    const unsigned long long key = own ? sh.akeys[lane] : ~0ull;
    const int r = own ? sel_key_r(key) - P.b_off : 0;
    const unsigned c = (unsigned)(key & 0xffffu);
    const int er = __shfl_sync(kFull, e, r);
    unsigned lt = 0u, same = 0u, clo = 0u;
    // all 32 key slots in one unrolled pass: the 16 broadcast 16-byte loads issue back to back,
    // the slots at or beyond nA masked off
    const ulonglong2* ak2 = reinterpret_cast<const ulonglong2*>(sh.akeys);
    const unsigned valid = nA >= 32 ? 0xffffffffu : ((1u << nA) - 1u);
#pragma unroll
    for (int j2 = 0; j2 < 16; ++j2) {
      const ulonglong2 pr = ak2[j2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const unsigned long long kj = u ? pr.y : pr.x;
        const unsigned bit = 1u << (2 * j2 + u);
        lt |= kj < key ? bit : 0u;
        same |= (((kj ^ key) >> 16) & 0xffffull) == 0ull ? bit : 0u;
        clo |= (unsigned)(kj & 0xffffu) < c ? bit : 0u;
      }
    }
    lt &= valid;
    same &= valid;
    clo &= valid;
    const bool elig = own && __popc(lt & same) < er;
    const unsigned Mq = __ballot_sync(kFull, elig);
    const int g = __popc(lt & Mq);
    if (elig) L.keys[g] = key;
    if (lane < bl) sh.a[lane] = 0;
    __syncwarp();
    stamp(P, lane == 0, 12);
    // ---- A5: tile 0 of the block path's scan over the sorted prefix ----
    const int ns = __popc(Mq);
    const bool act = lane < ns;
    const double bj = act ? (double)sel_key_b(L.keys[lane]) : 0.0;
    double incl = bj;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += u;
    }
    double excl = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) excl = 0.0;
    double before = 0.0;
    before += excl;
    const int ncut = __popc(__ballot_sync(kFull, act && bj > th_cut));
    const int narg = __popc(__ballot_sync(kFull, act && bj > th_arg));
    bool pass;
    if (P.selection == SMART_FROZEN) {
      pass = (L.ctab[0] > 0.0) ? (ac * bj * L.ctab[0] > rhs0 * L.dtab[0]) : (bj > 0.0);
    } else {
      const double C = L.ctab[lane];
      pass = (C > 0.0) ? (ac * bj * C > (rhs0 + P.c_T * before) * L.dtab[lane]) : (bj > 0.0);
    }
    const unsigned fail = __ballot_sync(kFull, lane < ncut && !pass);
    const int js = fail ? __ffs(fail) - 1 : ncut;
    stamp(P, lane == 0, 13);
    // ---- A6: per-request admits, next-frontier counts / offsets, entries, the flag ----
    const bool adm = elig && g < js;
    const unsigned A = __ballot_sync(kFull, adm);
    const int idx = __popc(same & clo & A);  // canonical order within the request
    if (adm) sh.a[r] = __popc(same & A);
    __syncwarp();
    const int a = lane < bl ? sh.a[lane] : 0;
    const bool fcond = st.fin || a == 0 || st.nd + a >= P.B;  // Alg.1 line 10
    const int nx = (lane < bl && !fcond) ? a : 0;
    int inx = nx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFull, inx, o);
      if (lane >= o) inx += u;
    }
    const int base = inx - nx, tot = __shfl_sync(kFull, inx, 31);
    // the row count first: the streaming CTAs take their team layout from it and then poll their
    // rows' self-validating entries, which follow
    if (lane == 0) pub(tot);
    const int basr = __shfl_sync(kFull, base, r), ndr = __shfl_sync(kFull, st.nd, r);
    const int nxr = __shfl_sync(kFull, nx, r), offr = __shfl_sync(kFull, st.off, r);
    stamp(P, lane == 0, 17);
    const int node = ndr + 1 + idx;
    const float bf = own ? sel_key_b(key) : 0.f;
    if (adm && nxr > 0) {
      const int pos = basr + idx;
      pub.entry(pos, r, node);
      Mn.fe[pos] = make_int2(r, node);  // the next layer's rows, kept in shared memory
      Mn.pc[pos] = bf;                  // NODE_SUM: b == cum
      Mn.slot[pos] = idx;
      fr_n[pos] = make_int2(r, node);
      frc_n[pos] = bf;
    }
    __syncwarp();
    stamp(P, lane == 0, 18);
    stamp(P, lane == 0, 19);
    // ---- after the flag: node records, per-request state, E, trace ----
    if (lane < bl) fro_n[lane] = base;
    if (lane == 0) *frt_n = tot;
    if (adm) {
      const int q = offr * k + (int)c;
      const int4 rec = crec[q];
      const size_t o = (size_t)r * T + node;
      P.tok[o] = rec.x;
      P.parent[o] = rec.w;
      P.depth[o] = layer;
      P.p[o] = __int_as_float(rec.y);
      P.cum[o] = __int_as_float(rec.z);
      P.cand_node[lbase + q] = node;
      P.cand_adm[lbase + q] = 1;
      L.cslot[r * L.wf + idx] = bf;
    }
    __syncwarp();
    if (lane < bl) {
      if (a > 0) {
        double esum = 0.0;  // canonical order
#pragma unroll 1
        for (int u = 0; u < a; ++u) esum += (double)L.cslot[lane * L.wf + u];
        st.E += esum;  // node sum (Q11)
        P.E_r[lane] = st.E;
      }
      const bool fnew = fcond && st.cnt > 0;
      if (fnew) P.finished[lane] = 1;
      P.n_nodes[lane] = st.nd + 1 + a;
      frn_n[lane] = nx;
      st.fin = st.fin || fnew;
      st.nd += a;
      st.cnt = nx;
      st.off = base;
      sh.nn[lane] = st.nd + 1;
    }
    if (layer == P.d || tot == 0) {
      // the trees are final: warp 0 publishes the verify rows ((request, node), request-major, as
      // self-validating entries) and their count right away, from its registers
      const int nr = lane < bl ? st.nd + 1 : 0;
      int vin = nr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(kFull, vin, o);
        if (lane >= o) vin += u;
      }
      const int voff = vin - nr, NR = __shfl_sync(kFull, vin, 31);
      const unsigned vtag = entry_tag(tag, 31);
      for (int j = 0; j < nr; ++j) {
        P.vrow_rn[voff + j] = make_int2(lane, j);
        st_relaxed_u64(&P.fr_tag[voff + j], ((unsigned long long)vtag << 32) | ((unsigned)lane << 10) | (unsigned)j);
      }
      if (lane < bl) P.vrow_off[lane] = voff;
      if (lane == 0) P.vrow_off[bl] = NR;
      __syncwarp();
      if (lane == 0) {
        st_relaxed_u64(&P.ctl->flag[kVerifySlot], ((unsigned long long)tag << 32) | (unsigned)(verify ? NR : 0));
        sh.vpub = 1;
      }
    }
    double Ea = lane < bl ? st.E : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Ea += __shfl_xor_sync(kFull, Ea, o);
    // argmax_j S_j over the prefixes up to narg (block path's association and tie rule): final
    // when narg == ne or the window is convex (th_arg > 0), else the full list (small_trace_full)
    auto sp = [&](double E, int j) {  // b*S at N0 + j (window)
      const double C = L.ctab[j];
      return C > 0.0 ? P.c_T * ((double)P.omega * bc + E) / C : 0.0;
    };
    double bestS = sp(E0, 0);
    int bestj = 0;
    if (lane < narg) {
      const double Sa = sp(E0 + before + bj, lane + 1);
      if (Sa > bestS) {
        bestS = Sa;
        bestj = lane + 1;
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
    const bool full = narg < ne && !(th_arg > 0.0);
    if (lane == 0) {
      DevTrace& tr = P.trace[layer - 1];
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
      tr.dc0 = L.dtab[0];
      tr.saturated = (N0 + ne >= P.sat_from) ? 1 : 0;
      if (tr.saturated) atomicOr(P.err, kErrSaturated);
      tr.select_path = full ? 2 : 1;
      tr.n_screened = nA;
      sh.N0next = N0 + js;
      sh.need_full = full ? 1 : 0;
    }
    stamp(P, lane == 0, 22);
  }
  consumer_sync();
  if (sh.need_full) {
    // the full sorted eligible list for argmax_j (rare): A3 inputs of this layer from the rows
    if (warp == 0 && lane < bl) L.base[lane] = eb;
    for (int rr = tid; rr < bl; rr += kConsumers) {
      L.cnt[rr] = 0;
      L.off[rr] = R;
    }
    consumer_sync();
    for (int row = tid; row < R; row += kConsumers) {
      const int rq = L.rreq[row];
      atomicAdd(&L.cnt[rq], 1);
      atomicMin(&L.off[rq], row);
    }
    consumer_sync();
    small_trace_full(P, dsm, sh, nct, ne, sh.E0, bc);
    if (tid == 0) P.trace[layer - 1].argmax_j = sh.bestj;
  }
  stamp(P, tid == 0, 16);
  return true;
}

template <bool BF16>
__device__ void select_role(const Params& P, char* dsm, size_t sel_bytes, const int32_t* root_tok,
                            const int32_t* root_pos, const StepOut& out, bool verify, unsigned tag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp >= kConsumerWarps) return;
  const int S = P.step_S, k = P.k, cpr = P.cpr, kp = list_stride(k), T = P.T, bl = P.b_loc;
  const int rows_cap = P.cap_rows > bl ? P.cap_rows : bl;
  MergeLayout M = merge_layout(dsm + a16(sel_bytes), rows_cap);
  // the small path's row descriptors by layer parity (select_small writes the next layer's)
  const MergeLayout Mb[2] = {M, merge_layout(dsm + a16(sel_bytes) + merge_bytes(rows_cap), rows_cap)};

  // ---- begin step: S_0 = A_0 = {root} for every request ----
  for (int r = tid; r < bl; r += kConsumers) {
    const size_t o = (size_t)r * T;
    P.n_nodes[r] = 1;
    P.tok[o] = root_tok ? root_tok[r] : -1;
    P.parent[o] = -1;
    P.depth[o] = 0;
    P.p[o] = 1.f;  // root: p = cum = 1
    P.cum[o] = 1.f;
    P.path_sum[o] = 0.0;
    P.E_r[r] = 0.0;
    P.leaf_cnt[r] = 1;
    P.leaf_sum[r] = 0.0;
    P.finished[r] = 0;
    P.root_pos[r] = root_pos ? root_pos[r] : 0;
    P.fr[0][r] = make_int2(r, 0);
    P.fr_cum[0][r] = 1.f;
    P.fr_cnt[0][r] = 1;
    P.fr_off[0][r] = r;
  }
  if (tid < SMART_MAX_DEPTH) {
    DevTrace t0{};
    P.trace[tid] = t0;
  }
  if (tid == 0) {
    *P.fr_total[0] = bl;
    *P.err = 0;
    P.sum_accept[0] = 0ull;
    P.sum_accept[1] = 0ull;
    *P.N_glob = 0;
    *P.E_glob = 0.0;
  }
  consumer_sync();
  // small batches: select_small with the per-request state in warp 0's registers
  const bool small = P.nranks == 1 && bl <= 32 && P.accept_model == SMART_NODE_SUM &&
                     (P.selection == SMART_PREFIX || P.selection == SMART_FROZEN) && P.debug_mode != 7;
  __shared__ SmallShared ssm;
  SmallState st;
  st.cnt = lane < bl ? 1 : 0;
  st.off = lane;
  st.nd = st.fin = 0;
  st.E = 0.0;
  bool rows_in_smem = false;  // layer 1: the roots, from the global frontier written above
  if (tid == 0) {
    ssm.N0next = 0;
    ssm.vpub = 0;
  }
  if (tid < bl && tid < 32) ssm.nn[tid] = 1;
  consumer_sync();

  for (int layer = 1; layer <= P.d; ++layer) {
    const int par = (layer - 1) & 1;
    const int R = *P.fr_total[par];
    if (R == 0) break;
    const int t = team_size(R, S, cpr);
    const size_t lbase = (size_t)(layer - 1) * P.cap_rows * k;
    bool staged = false;  // select_small fell back with the records staged
    auto wait_merge = [&](SelLayout& L, int4* crec) -> bool {
      if (staged) return true;
      // row descriptors (this CTA's own writes) while the rows stream
      for (int row = tid; row < R; row += kConsumers) {
        const int2 fe = P.fr[par][row];
        M.fe[row] = fe;
        M.pc[row] = P.fr_cum[par][row];
        M.slot[row] = row - P.fr_off[par][fe.x];
        L.rreq[row] = fe.x;
      }
      consumer_sync();
      if (tid == 0) pb_max(P, layer, kPbSync1);
      // the rows' merged candidates (team merges), polled as tagged lines straight into the
      // selection's staged records: cum = cum(parent) * p (Eq.(3)), parent = the row's node
      const unsigned lt = entry_tag(tag, layer);
      for (int q = tid; q < R * k; q += kConsumers) {
        const uint2 v = wait_line(P.seg_cand + q, lt, P.err);
        const int row = q / k;
        crec[q] = make_int4((int)v.x, (int)v.y, __float_as_int(__fmul_rn(M.pc[row], __uint_as_float(v.y))), M.fe[row].y);
      }
      consumer_sync();
      if (tid == 0) pb_max(P, layer, kPbMerged);
      return true;
    };
    bool done = false;
    if (small) {
      done = select_small(P, layer, R, dsm, Mb[layer & 1], Mb[(layer + 1) & 1], rows_in_smem, st, ssm, tag,
                          StepPub{&P, tag, layer}, verify);
      staged = !done;  // records and row requests are staged for the generic selection
      rows_in_smem = done;
    }
    if (!done) {
      select_layer<kConsumers>(P, layer, kSelFull, dsm, wait_merge, StepPub{&P, tag, layer});
      if (small) {
        consumer_sync();
        if (tid == 0) {
          P.trace[layer - 1].select_path = 3;
          P.trace[layer - 1].n_screened = ssm.n_above;
        }
        if (warp == 0) {
          small_state_load(P, layer & 1, lane, st);
          if (lane < bl) ssm.nn[lane] = st.nd + 1;
        }
        if (tid == 0) ssm.N0next = *P.N_glob;
      }
    }
    if (tid == 0) pb_max(P, layer, kPbPublished);
    consumer_sync();
    // inspection copies (smart_get_candidates) after the frontier is out: the candidate records
    // and each row's (request, slot), from the selection's staged records
    {
      const SelLayout L = sel_layout(dsm, bl, P.cap_rows * k, k, P.sort_cap);
      const int4* crec = reinterpret_cast<const int4*>(reinterpret_cast<const char*>(L.E) + sel_align((size_t)bl * 8) +
                                                       2 * (size_t)P.sort_cap * 8);
      int4* gc = reinterpret_cast<int4*>(P.cand + lbase);
      const MergeLayout& Mc = small ? Mb[layer & 1] : M;  // this layer's row descriptors
      for (int q = tid; q < R * k; q += kConsumers) {
        gc[q] = crec[q];
        P.cand_b[lbase + q] = L.cb[q];
      }
      for (int row = tid; row < R; row += kConsumers)
        P.cand_rs[(size_t)(layer - 1) * P.cap_rows + row] = make_int2(Mc.fe[row].x, Mc.slot[row]);
    }
    consumer_sync();  // the scratch is reused by the next layer's selection / the final phase
    if (tid == 0) pb_max(P, layer, kPbSelDone);
    if (SMART_PROBES && P.dbg && tid == 0)  // the selection's clock64 phase stamps of this layer
      for (int j = 9; j <= 22; ++j) P.dbg[3000 + layer * 16 + (j - 9)] = P.dbg[32 + j];
  }

  if (SMART_PROBES && P.dbg && tid == 0) P.dbg[1000] = gtime();
  // ---- verify rows first: (request, node) of every tree row, request-major (A8 reads all of
  // them), as self-validating tagged words (entry tag of layer 31) and the row count as a tagged
  // flag, plain stores: nothing else is needed before the target rows can stream ----
  int* s_n = reinterpret_cast<int*>(dsm);                // [bl + 1] node counts, [bl + 1] scan scratch
  int* s_par = s_n + a16((size_t)(2 * bl + 2) * 4) / 4;  // [bl * T] parent, depth, token, target argmax
  int* s_dep = s_par + (size_t)bl * T;
  int* s_tok = s_dep + (size_t)bl * T;
  int* s_arg = s_tok + (size_t)bl * T;
  int* s_off = s_n + bl + 1;  // exclusive scan of the node counts
  // node counts: from the small path's shared copy (no round trip through L2), else the global state
  for (int r = tid; r < bl; r += kConsumers) s_off[r] = s_n[r] = small ? ssm.nn[r] : P.n_nodes[r];
  consumer_sync();
  if (warp == 0) {
    const int tot = warp_excl_scan_smem(s_off, bl, lane);
    if (lane == 0) s_off[bl] = tot;
  }
  consumer_sync();
  const int NR = s_off[bl];
  const unsigned vtag = entry_tag(tag, 31);
  const bool vdone = small && ssm.vpub;  // already published by select_small's warp 0
  for (int e = tid; e < bl * T && !vdone; e += kConsumers) {
    const int r = e / T, j = e - r * T;
    if (j < s_n[r]) {
      P.vrow_rn[s_off[r] + j] = make_int2(r, j);
      st_relaxed_u64(&P.fr_tag[s_off[r] + j], ((unsigned long long)vtag << 32) | ((unsigned)r << 10) | (unsigned)j);
    }
  }
  for (int r = tid; r <= bl && !vdone; r += kConsumers) P.vrow_off[r] = s_off[r];
  if (tid == 0) {
    if (!vdone)
      st_relaxed_u64(&P.ctl->flag[kVerifySlot], ((unsigned long long)tag << 32) | (unsigned)(verify ? NR : 0));
    pb_max(P, kVerifySlot, kPbPublished);
  }
  if (SMART_PROBES && P.dbg && tid == 0) P.dbg[1001] = gtime();
  // ---- the final trees, staged in shared memory with one round of loads (this CTA's writes) ----
  for (int e = tid; e < bl * T; e += kConsumers) {
    s_par[e] = P.parent[e];
    s_dep[e] = P.depth[e];
    s_tok[e] = P.tok[e];
  }
  consumer_sync();
  if (SMART_PROBES && P.dbg && tid == 0) P.dbg[1002] = gtime();
  // ---- A7 while the target rows stream: ancestor-or-self bit rows, positions, parents, tokens ----
  const int MW = P.MW;
  for (int e = tid; e < bl * T; e += kConsumers) {
    const int r = e / T, j = e - r * T;
    const int n = s_n[r];
    const int* sp = s_par + (size_t)r * T;
    if (j < n) {
      if (out.mask) {
        for (int w = 0; w < MW; ++w) {
          uint32_t word = 0;
          for (int a = j; a >= 0; a = sp[a])  // ancestor-or-self chain (depth <= 16)
            if ((a >> 5) == w) word |= 1u << (a & 31);
          out.mask[(size_t)e * MW + w] = word;
        }
      }
      if (out.pos) out.pos[e] = P.root_pos[r] + s_dep[e];
      if (out.parent) out.parent[e] = sp[j];
      if (out.tok) out.tok[e] = s_tok[e];
    } else {
      if (out.mask)
        for (int w = 0; w < MW; ++w) out.mask[(size_t)e * MW + w] = 0u;
      if (out.pos) out.pos[e] = 0;
      if (out.parent) out.parent[e] = -1;
      if (out.tok) out.tok[e] = -1;
    }
  }
  for (int r = tid; r < bl && out.tree_len; r += kConsumers) out.tree_len[r] = s_n[r];
  // first child of every node (children of a node are contiguous in canonical order: a layer's
  // nodes are numbered by (frontier slot, rank)); -1 = leaf
  int* s_fc = s_arg + (size_t)bl * T;
  for (int e = tid; e < bl * T; e += kConsumers) s_fc[e] = -1;
  consumer_sync();
  for (int e = tid; e < bl * T; e += kConsumers) {
    const int r = e / T, j = e - r * T;
    if (j >= 1 && j < s_n[r]) {
      const int p = s_par[e];
      if (s_par[e - 1] != p || j == 1) s_fc[(size_t)r * T + p] = j;
    }
  }
  if (tid == 0) pb_max(P, kVerifySlot, kPbMerged);  // mask outputs written
  if (!verify || NR == 0) return;

  // ---- A8 walk once every verify slice has posted its row maxima ----
  {
    // every verify CTA's done word (polled in parallel; relaxed load + fence = acquire)
    const int want = range_ctas(NR * cpr, S, P.min_units);
    bool seen = false;
    for (int c = tid; c < want; c += kConsumers) {
      (void)wait_tag_relaxed(&P.ctl->vdone[c], tag, P.err);
      seen = true;
    }
    if (seen) fence_acq_rel_gpu();
  }
  consumer_sync();
  if (tid == 0) pb_max(P, kVerifySlot, kPbArrived);
  // every node, in parallel: the target's argmax token and the child holding it (-1: none; the
  // children of a node are contiguous in canonical order, sibling tokens distinct), so that the
  // walk below is a chain of single loads
  for (int e = tid; e < bl * T; e += kConsumers) {
    const int r = e / T, u = e - r * T, n = s_n[r];
    if (u < n) {
      unsigned long long* slot = P.vbest + e;
      const int tgt = (int)(0xffffffffu - (uint32_t)__ldcg(slot));
      *slot = 0ull;  // cleared for the next step
      s_arg[e] = tgt;
      const int* sp = s_par + (size_t)r * T;
      const int* stk = s_tok + (size_t)r * T;
      int nx = -1;
      for (int j = s_fc[e]; j >= 0 && j < n && sp[j] == u; ++j)
        if (stk[j] == tgt) {
          nx = j;
          break;
        }
      s_fc[e] = nx;  // (this thread's own entry: read above, not read by any other thread)
    }
  }
  consumer_sync();
  if (SMART_PROBES && P.dbg && tid == 0) P.dbg[1003] = gtime();
  const int D = P.d > 0 ? P.d : 1;
  unsigned long long accs = 0ull, nods = 0ull;
  for (int r = tid; r < bl; r += kConsumers) {
    const int n = s_n[r];
    const int* sa = s_arg + (size_t)r * T;
    const int* fc = s_fc + (size_t)r * T;
    int cur = 0, acc = 0, bon = -1;
    for (;;) {  // follow the child holding the target's argmax token, else stop
      const int found = fc[cur];  // that child, found above
      if (found < 0) {
        bon = sa[cur];
        break;
      }
      if (out.accept_path && acc < D) out.accept_path[(size_t)r * D + acc] = found;
      ++acc;
      cur = found;
    }
    if (out.accept_len) out.accept_len[r] = acc;
    if (out.bonus) out.bonus[r] = bon;
    if (out.accept_path)
      for (int j = acc; j < D; ++j) out.accept_path[(size_t)r * D + j] = -1;
    accs += (unsigned long long)acc;
    nods += (unsigned long long)(n - 1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    accs += __shfl_xor_sync(kFull, accs, o);
    nods += __shfl_xor_sync(kFull, nods, o);
  }
  if (lane == 0 && (accs || nods)) {
    atomicAdd(P.sum_accept, accs);
    atomicAdd(P.sum_accept + 1, nods);
  }
}

template <bool BF16>
__global__ void __launch_bounds__(kStepThreads, 2)
step_kernel(Params P, size_t sel_bytes, const char* __restrict__ draft, long long ld_d, const char* __restrict__ target,
            long long ld_t, const int32_t* root_tok, const int32_t* root_pos, StepOut out) {
  extern __shared__ __align__(128) char dsm[];
  __shared__ unsigned s_tag;
  const bool sel = (int)blockIdx.x == (int)gridDim.x - 1;
  if (!sel && threadIdx.x == 0) {
    StreamPipe& pipe = *reinterpret_cast<StreamPipe*>(dsm + kStages * kChunkBytes);
    StepShared& sh = *reinterpret_cast<StepShared*>(dsm + kStages * kChunkBytes + sizeof(StreamPipe));
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pipe.full[s], 1);
      mbar_init(&pipe.empty[s], kConsumerWarps);
    }
    for (int e = 0; e < SMART_MAX_DEPTH + 2; ++e) mbar_init(&sh.evb[e], 1);
    mbar_fence_init();
    sh.cs.tau = 0ull;
  }
  pdl_wait();  // the previous kernel of the stream (e.g. the previous step) has completed
  if (threadIdx.x == 0) s_tag = __ldcg(&P.ctl->epoch) + 1u;
  if (threadIdx.x == 0) pb_min(P, 0, kPbFlagMin);  // kernel start (earliest CTA)
  __syncthreads();
  const unsigned tag = s_tag;
  if (sel) select_role<BF16>(P, dsm, sel_bytes, root_tok, root_pos, out, target != nullptr, tag);
  else stream_role<BF16>(P, dsm, draft, ld_d, target, ld_t, tag);
  __syncthreads();
  if (threadIdx.x == 0) pb_max(P, 0, kPbSelDone);  // kernel end (latest CTA)
  pdl_trigger();
  if (threadIdx.x == 0) {
    if (atomicAdd(&P.ctl->exit_cnt, 1) == (int)gridDim.x - 1) {  // the last CTA: next launch's epoch
      P.ctl->exit_cnt = 0;
      P.ctl->epoch = tag;
    }
  }
}

}  // namespace

size_t step_stream_smem_bytes() { return (size_t)kStages * kChunkBytes + sizeof(StreamPipe) + sizeof(StepShared); }

size_t step_select_smem_bytes(const Params& P, int S, size_t sel_bytes) {
  const int rows_cap = P.cap_rows > P.b_loc ? P.cap_rows : P.b_loc;
  const size_t sel = a16(sel_bytes) + 2 * merge_bytes(rows_cap);
  const size_t fin = a16((size_t)(2 * P.b_loc + 2) * 4) + (size_t)5 * P.b_loc * P.T * 4;
  return sel > fin ? sel : fin;
}

// grid of the step kernel (all CTAs co-resident: grid = SMs x occupancy) and its dynamic shared
// memory (the larger of the streaming CTA's ring and the selection CTA's scratch); 0 if the
// selection scratch does not fit one CTA
int step_grid(const Params& P, size_t sel_bytes, size_t* smem_out) {
  int dev = 0, nsm = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, step_kernel<true>);
  const int lim = optin - (int)fa.sharedSizeBytes;  // dynamic + static <= the opt-in maximum
  for (int b = 0; b < 2; ++b) {
    cudaFuncSetAttribute(b ? step_kernel<true> : step_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    cudaFuncSetAttribute(b ? step_kernel<true> : step_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  }
  size_t smem = step_stream_smem_bytes();
  int grid = 0;
  for (int it = 0; it < 3; ++it) {
    int occ = 0;
    if (smem > (size_t)lim ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step_kernel<true>, kStepThreads, smem) != cudaSuccess ||
        occ < 1) {
      cudaGetLastError();
      return 0;
    }
    if (const char* o = getenv("SMART_STEP_OCC")) occ = std::max(1, std::min(occ, atoi(o)));  // experiments only
    grid = std::min(nsm * occ, kStepMaxGrid);
    const size_t need = std::max(step_stream_smem_bytes(), step_select_smem_bytes(P, grid - 1, sel_bytes));
    if (need <= smem) break;
    smem = need;  // fewer CTAs per SM: recompute the grid (the scratch shrinks with S)
  }
  *smem_out = smem;
  return grid;
}

void launch_step(const Params& P, int grid, size_t smem, size_t sel_bytes, const void* draft, long long ld_d,
                 const void* target, long long ld_t, const int32_t* root_tok, const int32_t* root_pos,
                 const StepOut& out, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  Params Q = P;
  Q.step_S = grid - 1;
  Q.sel_rec = 1;  // the row merge stages the candidate records in the selection's scratch
  const char* d = static_cast<const char*>(draft);
  const char* t = static_cast<const char*>(target);
  if (P.dtype == SMART_BF16)
    cudaLaunchKernelEx(&cfg, step_kernel<true>, Q, sel_bytes, d, ld_d, t, ld_t, root_tok, root_pos, out);
  else
    cudaLaunchKernelEx(&cfg, step_kernel<false>, Q, sel_bytes, d, ld_d, t, ld_t, root_tok, root_pos, out);
}

}  // namespace smart
