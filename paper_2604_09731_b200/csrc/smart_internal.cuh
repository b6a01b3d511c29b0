// smart_internal.cuh — device-side layout and helpers of libsmart (B200, sm_100a).
//
// Everything here is product code; it shares nothing with oracle/ (the fp64 test oracle).
// Citations: P:n = PAPER.md line n (arXiv 2604.09731); Q# = DESIGN.md §3 reading.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "smart.h"

namespace smart {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kChunkBytes = 16384;       // streamed unit of a logit row (16 KiB)
constexpr int kStreamThreads = 256;      // CTA size of the streaming kernels (8 warps)
constexpr int kStreamWarps = kStreamThreads / kWarp;
constexpr int kVecPerThread = kChunkBytes / 16 / kStreamThreads;  // 4 x 16 B per thread
constexpr int kWarpBuf = 64;             // per-warp candidate staging (top-k filter)
constexpr int kSegBuf = 128;             // per-warp segment candidate buffer
constexpr int kSelectThreads = 1024;     // single-CTA selection kernel
constexpr int kMaxK = 32;
constexpr int kMaxCpr = 64;   // chunks per row (V*esz <= 1 MiB)
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kIdxSentinel = 0x7fffffff;
constexpr int kStageRows = 64;  // row descriptors a streaming CTA stages in shared memory

// error flag bits (smart_stats.error_flags)
constexpr int kErrDraftNaN = 1;
constexpr int kErrTargetNaN = 2;
constexpr int kErrSaturated = 4;
constexpr int kErrTimeout = 8;   // a device-side wait gave up (broken launch sequence); sticky

// one candidate produced by A1/A2 for (frontier row, rank j)
struct Cand {
  int32_t tok;
  float p;
  float cum;
  int32_t parent;  // node index of the expanded frontier node
};

// control block of the persistent whole-step kernel (step.cu), in the workspace (zeroed at
// create).  Flags carry (tag << 32 | value) with tag = epoch + 1 of the launch, so a step never
// sees a previous step's flags and nothing needs resetting between steps; the last CTA to exit
// advances the epoch.
constexpr int kVerifySlot = SMART_MAX_DEPTH + 1;
constexpr int kStepMaxGrid = 512;  // persistent step kernel: CTAs per launch at most
struct StepCtl {
  unsigned long long flag[SMART_MAX_DEPTH + 2];  // [l]: layer-l frontier rows published; [kVerifySlot]: verify rows
  unsigned long long vdone[kStepMaxGrid];        // [s]: streaming CTA s posted its verify row maxima (tag)
  int exit_cnt;
  unsigned epoch;
};

// device copy of one layer's trace (same fields as smart_layer_trace)
struct DevTrace {
  int32_t executed, n_rows, n_cand, n_elig, n_admit, argmax_j, N0, saturated, select_path, n_screened;
  double E0, S0, S_after, dc0;
};

// Everything a kernel needs: config scalars + workspace pointers.  Passed by value.
struct Params {
  // ---- config ----
  int V, k, d, Wq, b_loc, b_glob, b_off, B, T, MW;
  int selection, accept_model, marginal, cost_scope, dtype, row_mode, omega;
  int esz;            // bytes per logit
  int chunk_elems;    // elements per 16 KiB chunk
  int cpr;            // chunks per row
  int cap_rows;       // frontier rows per layer (local)
  int nranks, rank;
  double alpha, lambda, beta, gamma, delta, rho, eta, c_T;

  // ---- per-request tree state [b_loc] / [b_loc*T] ----
  int* n_nodes;       // incl. root
  int* tok;
  int* parent;
  int* depth;
  float* p;
  float* cum;
  double* path_sum;   // PATH_MEAN: sum of cum on root->node path
  double* E_r;        // acceptance estimate of request r (Q11)
  int* leaf_cnt;      // |P_r|
  double* leaf_sum;   // sum over leaves of path_sum
  int* finished;
  int* root_pos;

  // ---- frontier, ping-pong by layer parity ----
  int2* fr[2];        // (local request, node)
  float* fr_cum[2];   // cum of each frontier node (prefetched by the row merge)
  int* fr_cnt[2];     // [b_loc]
  int* fr_off[2];     // [b_loc] exclusive prefix
  int* fr_total[2];   // [1]

  // ---- A1 streaming scratch ----
  int* layer_done;    // [SMART_MAX_DEPTH] rows merged per layer (self-resetting)
  int* fr_ready;      // [SMART_MAX_DEPTH + 1] frontier of layer l published (reset by begin_step)
  Cand* cand;         // [d][cap_rows*k]
  float* cand_b;      // [d][cap_rows*k] benefit
  int* cand_adm;      // [d][cap_rows*k] admitted flag
  int* cand_node;     // [d][cap_rows*k] node index of an admitted candidate (BASELINE rerank)
  int2* cand_rs;      // [d][cap_rows] (local request, frontier slot) of each candidate row

  // ---- cost model tables (fp64, host-built with the same formula; N in [0, n_cost)) ----
  const double* cost_tab;   // cost(N) = C_draft(N) + C_verify(N)         Eqs.(4),(5)
  const double* dc_tab;     // marginal cost at N (DERIVATIVE Eq.(15) / DIFFERENCE)
  int n_cost;
  int sort_cap;             // key capacity of the selection sort (power of two)
  int sel_rec;              // 1: the selection stages the layer's candidate records in smem
  int min_units;            // chunks per CTA at least in the streaming kernels
  long long sat_from;       // smallest N whose exponent was clamped (Q17)

  // ---- optional timing probes (SMART_TIMING=1): globaltimer ns, see probe() ----
  unsigned long long* dbg;
  int debug_mode;     // SMART_DEBUG_MODE (timing experiments only; 0 in production)

  // ---- select / stats ----
  DevTrace* trace;    // [SMART_MAX_DEPTH]
  int* err;           // [1]
  unsigned long long* sum_accept;  // [2]: sum of accept lengths, sum of drafted nodes (local)
  unsigned long long* sum_glob;    // [2]: the same over all ranks (C2 all-reduce; = local on one rank)
  double* E_glob;     // [1] sum_r E_r after the last select
  int* N_glob;        // [1]

  // ---- verify scratch ----
  int* vrow_off;      // [b_loc+1]
  int2* vrow_rn;      // [b_loc*T] (request, node) of each verify row (written by the mask kernel)
  unsigned long long* vbest;  // [b_loc*T] target argmax key of each tree row (red.max; cleared by the walk)

  // ---- persistent whole-step kernel (step.cu) ----
  // self-validating 16-byte lines {a, tag, b, tag} (tag = entry tag of the launch and layer):
  uint4* seg_key;   // slice top-k lists of the current layer, [row * t + member][k] (key lo, key hi)
  uint4* seg_ms;    // per-chunk softmax partials of the current layer, [row][cpr] (M_c, S_c)
  uint4* seg_cand;  // the merged candidates of the current layer, [row][k] (token, p)
  StepCtl* ctl;
  unsigned long long* fr_tag;    // [max(cap_rows, b_loc * T)] self-validating frontier entries
                                 // ((tag << 5 | layer) << 32) | r << 10 | node; then the verify rows (layer 31)
  int step_S;                    // streaming CTAs (the grid's last CTA runs the selection)

  // ---- multi-rank exchange (select phase 0 -> NCCL all-gather -> select phase 1) ----
  // per-rank record: keys[m_cap] u64 | E_r[b_loc] f64 | hdr[b_loc] n_r, hdr[b_loc] = count
  int m_cap;
  long long xstride;  // bytes per rank record
  char* xs;           // send record
  char* xr;           // [nranks] gathered records (peer exchange: this rank's receive buffer)
  // peer exchange (smart_attach_peer_exchange): every rank's receive buffer as seen from here, the
  // byte offset of the per-rank tag words in a receive buffer, and the step counter of the tags
  char* const* xpeer;
  long long xtag_off;
  unsigned long long xepoch;
};

// ------------------------------------------------------------------------------------------
// small device helpers
// ------------------------------------------------------------------------------------------

// order of A1 top-k and of the verify argmax: larger value, then lower index (Q9)
__device__ __forceinline__ bool better(float av, int ai, float bv, int bi) {
  return av > bv || (av == bv && ai < bi);
}

// release/acquire fences at GPU scope (cheaper than the sequentially consistent __threadfence)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// arrival counter: one thread, after a CTA barrier, publishes the CTA's writes (release, cumulative
// over the barrier) and acquires the other arrivals' writes (CUTLASS-semaphore pattern)
__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// fire-and-forget arrival with release semantics, and the matching acquire poll
__device__ __forceinline__ void red_add_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// 64-bit top-k key: larger key = better (value desc, then index asc) — one compare per step
__device__ __forceinline__ unsigned long long tk_key(float v, int i);
__device__ __forceinline__ float tk_val(unsigned long long key);
__device__ __forceinline__ int tk_idx(unsigned long long key);

// packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2): two lanes of work per instruction
__device__ __forceinline__ unsigned long long f2pk(float a, float b) {
  return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}
__device__ __forceinline__ float f2lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t float_orderable(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ unsigned long long tk_key(float v, int i) {
  return ((unsigned long long)float_orderable(v) << 32) | (unsigned long long)(0xffffffffu - (unsigned)i);
}
__device__ __forceinline__ float tk_val(unsigned long long key) {
  const uint32_t o = (uint32_t)(key >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ int tk_idx(unsigned long long key) { return (int)(0xffffffffu - (uint32_t)key); }
constexpr unsigned long long kKeySentinel = 0x007fffff80000000ull;  // tk_key(-inf, INT_MAX)

// one-instruction warp max (sm_100a redux.sync .f32; NaN inputs ignored like fmaxf)
__device__ __forceinline__ float warp_max_fast(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// frontier-ready flag: one thread publishes after a CTA barrier (release, cumulative over the
// barrier); pollers acquire.  A poll that has not completed after ~2^31 tries (minutes: far beyond
// any time slicing or preemption) gives up and sets the sticky kErrTimeout flag, which
// smart_get_stats reports as SMART_EDEVICE; the context is not killed (no trap).
__device__ __forceinline__ void publish_flag(int* f) {
  asm volatile("st.release.gpu.global.s32 [%0], 1;" ::"l"(f) : "memory");
}
__device__ __forceinline__ bool wait_flag(const int* f, int* err) {
  for (unsigned it = 0; ld_acquire_gpu(f) == 0; ++it) {
    if (it > (1u << 31)) {
      atomicOr(err, kErrTimeout);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// Programmatic dependent launch: every kernel of the step is launched with programmatic stream
// serialization, runs its shared-memory prologue, then waits for the previous kernel of the
// stream (griddepcontrol.wait: full completion + memory visibility) before its first global read,
// and immediately lets the next kernel launch (its CTAs take resources as ours retire).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // api.cu: off with SMART_NO_PDL=1

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// probe slots: 0 min CTA start, 1 max CTA start, 2 max stream end, 3 last merge start,
// 4 last merge end, 5 select start, 6 select end, 7 max CTA end, 8 first merge start
// Probes are compiled in only with -DSMART_PROBES=1 (`SMART_PROBES=1 python -m
// paper_2604_09731_b200._build --force`): in the product build they cost nothing in the hot loops.
#ifndef SMART_PROBES
#define SMART_PROBES 0
#endif
__device__ __forceinline__ void probe_min(const Params& P, int slot) {
  if (SMART_PROBES && P.dbg) atomicMin(&P.dbg[slot], gtime());
}
__device__ __forceinline__ void probe_max(const Params& P, int slot) {
  if (SMART_PROBES && P.dbg) atomicMax(&P.dbg[slot], gtime());
}
// kernel timeline (dbg[64 + 2*kid] = min start, dbg[65 + 2*kid] = max end); kid: 0 begin,
// 1..d layer kernels, 20 mask, 21 verify, 22 select kernel; kid + 32: CTA launch (before the
// dependency wait)
__device__ __forceinline__ void tl_start(const Params& P, int kid) {
  if (SMART_PROBES && P.dbg && threadIdx.x == 0) atomicMin(&P.dbg[64 + 2 * kid], gtime());
}
__device__ __forceinline__ void tl_end(const Params& P, int kid) {
  if (SMART_PROBES && P.dbg && threadIdx.x == 0) atomicMax(&P.dbg[65 + 2 * kid], gtime());
}
// globaltimer stamp of one thread into dbg[slot] (slots 16..31: CTA 0 timeline)
__device__ __forceinline__ void gstamp(const Params& P, bool on, int slot) {
  if (SMART_PROBES && P.dbg && on) P.dbg[slot] = gtime();
}
// cycle stamps (clock64) of one thread into dbg[32 + slot]
__device__ __forceinline__ void stamp(const Params& P, bool on, int slot) {
  if (SMART_PROBES && P.dbg && on) P.dbg[32 + slot] = clock64();
}

// ---- cost model (fp64; Eqs.(4),(5),(15); clamp Q17) ----
__device__ __forceinline__ double cost_spec(const Params& P, double N, int* sat) {
  double a = P.delta * pow(N, P.rho);
  if (a > 700.0) { a = 700.0; *sat = 1; }
  return P.lambda * N + P.beta + P.gamma * (exp(a) - 1.0) + P.eta;
}
__device__ __forceinline__ double marginal_cost(const Params& P, long long N, int* sat) {
  if (P.marginal == SMART_DIFFERENCE) return cost_spec(P, (double)(N + 1), sat) - cost_spec(P, (double)N, sat);
  double M = (double)(N < 1 ? 1 : N);
  double a = P.delta * pow(M, P.rho);
  if (a > 700.0) { a = 700.0; *sat = 1; }
  return P.lambda + P.gamma * P.delta * P.rho * pow(M, P.rho - 1.0) * exp(a);
}
// b * S: c_T*(omega*b + E)/cost(N); 0/0 := 0 (Q4)
__device__ __forceinline__ double speed_b(const Params& P, double E, long long N, int b, int* sat) {
  double C = cost_spec(P, (double)N, sat);
  if (C <= 0.0) return 0.0;
  return P.c_T * ((double)P.omega * b + E) / C;
}

// ---- kernels (host launchers in api.cu) ----
__global__ void begin_step_kernel(Params P, const int32_t* root_tok, const int32_t* root_pos);
void launch_expand(const Params& P, int layer, const void* logits, long long ld_bytes, bool tma,
                   bool fuse_select, bool early, int grid, cudaStream_t s);
size_t layer_smem_bytes(int cpr, int k);
int expand_grid(int cpr, int k);
void launch_select(const Params& P, int layer, int phase, size_t smem, cudaStream_t s);
void launch_peer_push(const Params& P, int layer, cudaStream_t s);
void launch_peer_wait(const Params& P, int layer, cudaStream_t s);
size_t select_smem_bytes(int b_loc, int b_all, int sort_cap, int nc_cap, int nranks, int k);
size_t select_rec_bytes(int nc_cap);
cudaError_t select_set_smem(size_t bytes);
void launch_rerank(const Params& P, cudaStream_t s);
cudaError_t rerank_set_smem(size_t bytes);
size_t rerank_smem_bytes(const Params& P);
void launch_mask(const Params& P, uint32_t* mask, int32_t* pos, int32_t* parent, int32_t* tok,
                 int32_t* tree_len, cudaStream_t s);
void launch_verify(const Params& P, const void* target, long long ld_bytes, bool tma,
                   int32_t* accept_len, int32_t* accept_path, int32_t* bonus, int grid, cudaStream_t s,
                   bool sample = false, float inv_tau = 1.f, unsigned long long seed = 0ull);
size_t verify_smem_bytes(int T);
size_t walk_smem_bytes(int T);
cudaError_t walk_set_smem_bytes(size_t bytes);
int verify_occupancy(bool sample = false);
cudaError_t mask_set_smem_bytes(size_t bytes);
size_t mask_smem_bytes(int T, int b);
struct StepOut {
  uint32_t* mask;
  int32_t *pos, *parent, *tok, *tree_len, *accept_len, *accept_path, *bonus;
};
// persistent whole-step kernel (step.cu); sel_bytes = select_layer scratch incl. staged records
int step_grid(const Params& P, size_t sel_bytes, size_t* smem_out);  // 0: the config does not fit
size_t step_stream_smem_bytes();
size_t step_select_smem_bytes(const Params& P, int S, size_t sel_bytes);
void launch_step(const Params& P, int grid, size_t smem, size_t sel_bytes, const void* draft, long long ld_d,
                 const void* target, long long ld_t, const int32_t* root_tok, const int32_t* root_pos,
                 const StepOut& out, cudaStream_t s);
void launch_export_frontier(const Params& P, int parity, int32_t* d_frontier, int32_t* d_count,
                            cudaStream_t s);

}  // namespace smart
