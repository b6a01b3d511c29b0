/*
 * smart.h — C-ABI of the B200-native SMART hot path (libsmart.so).
 *
 * SMART (arXiv 2604.09731, "When is it Actually Worth Expanding a Speculative Tree?")
 * builds a speculative draft tree layer by layer, expanding a candidate only when its
 * marginal benefit/cost ratio beats the tree-level speedup (Eq.(16), PAPER.md P:347-355;
 * Algorithm 1), then verifies the tree with one target forward.  This library
 * is the data-parallel hot path of that controller for a batch of requests:
 *
 *   smart_begin_step       roots S_0 = A_0 = {root}
 *   smart_expand_step  A1  top-k + softmax of every frontier row
 *                      A2  path score cum = cum(parent) * p                (Eq.(3))
 *   smart_select       A3  marginal benefit b = cum/|P_r| (or cum), per-request budget
 *                          min(B - n_r, W)                                 (Eq.(13), Eq.(8))
 *                      A4  batch-global ranking (b desc, request asc, candidate asc)
 *                      A5  prefix scan + rule alpha*c_T*b/dc > S           (Eqs.(1),(12),(15),(16))
 *                      A6  commit A_l, S_l = S_{l-1} ∪ A_l, next frontier   (Eq.(7))
 *   smart_build_mask   A7  ancestor mask, position ids, parent indices, tokens
 *   smart_verify_accept A8 greedy (T=0) longest-accepted-path walk on target logits
 *   smart_verify_sample    A8 at temperature T > 0 (NEXT #1; P:453 reports T in {0, 1})
 *
 * Readings of the paper where it is silent or ambiguous are listed in DESIGN.md §3 (Q1..);
 * they are shared with the fp64 oracle in oracle/ (which this library never links).
 *
 * Conventions
 *  - All d_* pointers are DEVICE pointers owned by the caller.  The library never frees or
 *    retains them past completion of the work enqueued on `stream`.
 *  - `stream` is a cudaStream_t passed as void*.  Every step call is asynchronous, never
 *    synchronises the host, never allocates, and is legal inside CUDA-graph capture.
 *    Exception: smart_get_* calls synchronise the context's last stream.
 *  - One context serves one stream at a time; contexts are independent.
 *  - Host-side validation errors return synchronously (message in smart_last_error).
 *    Device-side anomalies (NaN/+inf logits, cost-exponent saturation) set sticky flags read
 *    by smart_get_stats; the step keeps running (saturated marginal costs never admit).
 *  - Logit rows: `vocab` entries, row stride `ld` ELEMENTS (ld >= vocab), dtype per config.
 *    Rows whose start is 16-byte aligned use 128-bit loads; others a scalar path.
 */
#ifndef SMART_H
#define SMART_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SMART_OK = 0,
  SMART_EINVAL = 1,    /* bad argument / config (see smart_last_error)            */
  SMART_ECUDA = 2,     /* CUDA runtime error                                       */
  SMART_ENCCL = 3,     /* NCCL error or NCCL library not loadable                  */
  SMART_ECAPACITY = 4, /* config exceeds compiled capacity                         */
  SMART_EDEVICE = 5,   /* sticky device flag set (NaN/+inf logits)                 */
  SMART_ESTATE = 6     /* call out of order (e.g. select before expand)            */
} smart_status;

typedef enum { SMART_BF16 = 0, SMART_FP32 = 1 } smart_dtype;
/* PREFIX / FROZEN: SMART's rule (Q7).  BASELINE (NEXT #3, Q32): the likelihood-maximising
 * two-stage policy of EAGLE-3 / MSD (Fig. 2(a)(b)): every layer expands the request's top-
 * max_frontier candidates by cum (no cost model); smart_build_mask first reranks all generated
 * candidates and keeps the top floor(budget_verify / batch) by cum (ancestor-closed by
 * construction).  BASELINE needs max_frontier >= 1 and a single rank (batch_local == batch_global). */
typedef enum { SMART_PREFIX = 0, SMART_FROZEN = 1, SMART_BASELINE = 2 } smart_selection;
typedef enum { SMART_NODE_SUM = 0, SMART_PATH_MEAN = 1 } smart_accept_model;  /* Q11 */
typedef enum { SMART_DERIVATIVE = 0, SMART_DIFFERENCE = 1 } smart_marginal;   /* Q5  */
typedef enum { SMART_COST_GLOBAL = 0, SMART_COST_LOCAL = 1 } smart_cost_scope;/* Q13 */
/* Row addressing of draft logits passed to smart_expand_step:
 *  FRONTIER: row i of d_logits belongs to frontier entry i (request-major, canonical order),
 *            i.e. what a real draft forward over the packed frontier produces.
 *  NODE:     row (r, u) lives at d_logits + (r*tree_capacity + u)*ld: one pool per step,
 *            each node's row read when that node is expanded (bench / test layout).
 *  POSITION: DFLASH (NEXT #4): one non-autoregressive draft forward gives
 *            max_depth independent position distributions per request; every frontier node of
 *            local request r at layer l expands with row d_logits + (r*max_depth + l-1)*ld
 *            (pool [batch_local, max_depth, ld], passed to every smart_expand_step).  With
 *            selection BASELINE and max_frontier >= floor(budget_verify / batch) this is the
 *            paper's Cartesian product of per-position top-k pruned to the top-g by cum; with
 *            PREFIX / FROZEN it is DFLASH+SMART. */
typedef enum { SMART_ROWS_FRONTIER = 0, SMART_ROWS_NODE = 1, SMART_ROWS_POSITION = 2 } smart_row_mode;

/* Cost-model constants (milliseconds): Eq.(4) C_draft = lambda*N + beta;
 * Eq.(5) C_verify = gamma*(exp(delta*N^rho)-1) + eta; Eq.(1) c_T = per-step AR cost. */
typedef struct {
  double lambda, beta, gamma, delta, rho, eta, c_T;
} smart_cost;

typedef struct {
  int32_t vocab;          /* V, 2 .. 2^24                                                  */
  int32_t top_k;          /* k, 1 .. min(V, 32)                                             */
  int32_t max_depth;      /* d, 0 .. 16                                                     */
  int32_t max_frontier;   /* W, nodes admitted per request per layer; 0 = unlimited (Q12)  */
  int32_t batch_local;    /* requests owned by this context (rank)                         */
  int32_t batch_global;   /* b, requests across all ranks; B = floor(budget_verify / b)    */
  int32_t batch_offset;   /* first global request owned: [offset, offset + local)         */
  int32_t budget_verify;  /* B_verify                                        */
  double alpha;           /* discount factor, (0, 1] (Eq.(12); default 0.8)          */
  int32_t bonus;          /* omega in S = c_T*(omega*b + E)/(b*cost(N)) (Q19), 0 or 1       */
  int32_t selection;      /* smart_selection                                                */
  int32_t accept_model;   /* smart_accept_model                                             */
  int32_t marginal;       /* smart_marginal                                                 */
  int32_t cost_scope;     /* smart_cost_scope                                               */
  int32_t logits_dtype;   /* smart_dtype (draft and target logits)                          */
  int32_t row_mode;       /* smart_row_mode                                                 */
  int32_t tree_capacity;  /* T: nodes per request incl. root; 0 = 1 + min(B, d*W)           */
                          /* (BASELINE: 0 = 1 + max(B, d*W))                                */
} smart_config;

typedef struct smart_ctx smart_ctx;

/* Derived sizes for a config (host-only, no device needed). */
typedef struct {
  int32_t B;              /* per-request budget floor(B_verify / b)                        */
  int32_t T;              /* tree capacity per request (incl. root)                        */
  int32_t mask_words;     /* ceil(T/32): u32 words per mask row                            */
  int32_t frontier_cap;   /* max frontier rows per layer on this rank                      */
  int32_t chunk_elems;    /* elements per streamed 16 KiB chunk                            */
} smart_sizes;

#define SMART_MAX_DEPTH 16

/* Per-layer trace, filled by smart_select (read with smart_get_stats). */
typedef struct {
  int32_t executed;       /* 1 if the layer had frontier rows                              */
  int32_t n_rows;         /* frontier rows expanded (local)                                 */
  int32_t n_cand;         /* candidates generated (local)                                   */
  int32_t n_elig;         /* eligible after per-request budget/W truncation (global)       */
  int32_t n_admit;        /* admitted (global) = first-failure cut j*                       */
  int32_t argmax_j;       /* argmax_j S_j over prefixes (reported, Q7)                      */
  int32_t N0;             /* drafted nodes before the layer (global)                        */
  int32_t saturated;      /* cost exponent clamped (Q17)                                    */
  int32_t select_path;    /* which selection ran (diagnostic): 0 the block selection, 1 the
                             small-batch one-warp path, 2 the same with the full sorted list
                             rebuilt for argmax_j, 3 the small path handed over to the block one */
  int32_t n_screened;     /* small-batch path: candidates above its benefit threshold (the
                             only ones ranked); 0 on the block path         */
  double E0;              /* sum_r E_r before the layer (global request order)              */
  double S0;              /* S before the layer (per request, Eq.(1) generalised)           */
  double S_after;         /* S after the layer                                              */
  double dc0;             /* marginal cost at N0                                            */
} smart_layer_trace;

typedef struct {
  int32_t layers_executed;
  int32_t error_flags;    /* bit0: NaN/+inf/all--inf draft row; bit1: NaN target row;
                             bit2: cost saturation seen; bit3: a device-side wait timed out
                             (calls out of order / a broken launch sequence)               */
  int64_t nodes_local;    /* sum over local requests of drafted nodes                      */
  int64_t accepted_local; /* sum of accept lengths (after smart_verify_accept)              */
  int64_t accepted_global;/* sum of accept lengths over all ranks (C2: one NCCL all-reduce at */
  int64_t nodes_global;   /* the end of verify when a communicator is attached; else local)  */
  int32_t step_kernel_grid; /* CTAs of the persistent whole-step kernel smart_run_step used for  */
  int32_t reserved;         /* the last step (0: the per-layer kernels ran)                    */
  double E_global, S_final;
  smart_layer_trace layer[SMART_MAX_DEPTH];
} smart_stats;

/* ---- lifecycle ------------------------------------------------------------------------ */

smart_status smart_query_sizes(const smart_config* cfg, smart_sizes* out);

/* Create a context on `device`, allocate all device workspace (sized from cfg caps). */
smart_status smart_create(const smart_config* cfg, const smart_cost* cost, int device,
                          smart_ctx** out);

/* Multi-GPU (cost_scope GLOBAL over several ranks): rank 0 calls smart_nccl_unique_id,
 * broadcasts the 128 bytes (e.g. via torch.distributed), then every rank calls
 * smart_attach_nccl.  libnccl.so.2 is loaded with dlopen on first use. */
smart_status smart_nccl_unique_id(uint8_t id_out[128]);
smart_status smart_attach_nccl(smart_ctx* ctx, const uint8_t id[128], int rank, int nranks);

/* Bring-your-own all-gather (no NCCL inside the library).  Each rank owns a send record of
 * smart_exchange_record_bytes() bytes and a receive buffer of nranks records (both device
 * memory, caller-owned, 256-byte aligned).  After smart_attach_exchange, smart_select(layer) runs
 * only the local phase (per-request eligibility, local sort) and fills d_send; the caller
 * all-gathers the records of all ranks in rank order into every rank's d_recv (e.g.
 * torch.distributed.all_gather_into_tensor on the same stream) and then calls
 * smart_select_finish(layer): merge of the gathered lists, the batch-global rule, commit of
 * this rank's requests.  Sharding: equal contiguous ranges, batch_offset = rank*batch_local. */
smart_status smart_exchange_record_bytes(const smart_config* cfg, int nranks, int64_t* bytes);
smart_status smart_attach_exchange(smart_ctx* ctx, int rank, int nranks, void* d_send, void* d_recv);
smart_status smart_select_finish(smart_ctx* ctx, int32_t layer, int32_t* d_frontier,
                                 int32_t* d_frontier_count, void* stream);

/* Peer exchange (NEXT #4; the per-layer exchange without a collective call).
 * Every rank owns one receive buffer of smart_peer_exchange_bytes() bytes (device memory,
 * 256-byte aligned, zeroed once by its owner): nranks records of smart_exchange_record_bytes()
 * bytes, then one 8-byte tag word per rank.  d_recv_bufs[g] is rank g's buffer as seen from this
 * process -- the same device pointers in one process, cudaIpcOpenMemHandle mappings across
 * processes (smart_ipc_get_handle / smart_ipc_open_handle; peer access over NVLink).  After
 * smart_attach_peer_exchange, smart_select(layer) runs the local phase and writes its record
 * straight into every rank's buffer (slot `rank`), then the tag word (step counter << 32 | layer)
 * with release semantics at system scope; smart_select_finish(layer) polls the nranks tag words of
 * its own buffer (acquire; a sticky SMART_EDEVICE timeout flag instead of a hang) and runs the
 * global phase.  Decisions are the same bits as with the all-gather.  smart_run_step drives both
 * halves per layer (on separate GPUs; ranks sharing one GPU must call them in lockstep, all local
 * phases before any finish).  Sharding as for smart_attach_exchange. */
smart_status smart_peer_exchange_bytes(const smart_config* cfg, int nranks, int64_t* bytes);
smart_status smart_attach_peer_exchange(smart_ctx* ctx, int rank, int nranks, void* const* d_recv_bufs);
/* CUDA IPC of a device allocation: 64-byte handle out, mapping in (this process), unmapping. */
smart_status smart_ipc_get_handle(void* d_ptr, uint8_t handle[64]);
smart_status smart_ipc_open_handle(const uint8_t handle[64], void** d_ptr);
smart_status smart_ipc_close(void* d_ptr);

smart_status smart_destroy(smart_ctx* ctx);

/* ---- one decode step -------------------------------------------------------------------- */

/* Reset the per-request trees: node 0 = root with token d_root_tok[r] (may be NULL -> -1)
 * and position d_root_pos[r] (may be NULL -> 0), p = cum = 1.  Frontier = all roots. */
smart_status smart_begin_step(smart_ctx* ctx, const int32_t* d_root_tok, const int32_t* d_root_pos,
                              void* stream);

/* A1+A2 for `layer` (1-based, in order).  Reads only the first frontier-count rows
 * (device-side count) of d_logits (row addressing per cfg.row_mode). */
smart_status smart_expand_step(smart_ctx* ctx, int32_t layer, const void* d_logits, int64_t ld,
                               void* stream);

/* A3-A6 for `layer`.  Optionally copies the next frontier out: d_frontier [frontier_cap][2]
 * int32 (local request, node index) and d_frontier_count [1]; either may be NULL. */
smart_status smart_select(smart_ctx* ctx, int32_t layer, int32_t* d_frontier,
                          int32_t* d_frontier_count, void* stream);

/* A7: d_mask [batch_local][T][mask_words] u32 (bit j of row i set iff node j is an ancestor-
 * or-self of node i), d_pos/d_parent/d_tok [batch_local][T] int32 (padding rows: 0/-1/-1),
 * d_tree_len [batch_local].  Any output may be NULL. */
smart_status smart_build_mask(smart_ctx* ctx, uint32_t* d_mask, int32_t* d_pos, int32_t* d_parent,
                              int32_t* d_tok, int32_t* d_tree_len, void* stream);

/* A8: greedy walk.  d_target row (r, node i) at d_target + (r*T + i)*ld; rows i >= tree_len
 * are never read.  Outputs: d_accept_len [batch_local], d_accept_path [batch_local][max(d,1)]
 * (node indices, -1 padded), d_bonus [batch_local].  Must follow smart_build_mask. */
smart_status smart_verify_accept(smart_ctx* ctx, const void* d_target, int64_t ld,
                                 int32_t* d_accept_len, int32_t* d_accept_path, int32_t* d_bonus,
                                 void* stream);

/* A8 at temperature `temperature` > 0 (reading Q31): at every
 * visited node one target token is drawn from softmax(logits / temperature) by Gumbel-max,
 *   argmax_v  logit_v / temperature - ln(-ln U_v),
 *   U_v = ((h >> 9) + 1/2) / 2^23,  h = lowbias32(rk + v * 0x9e3779b9) (mod 2^32),
 *   rk = high half of SplitMix64(seed + ((batch_offset + r) << 22 | node) * 0x9e3779b97f4a7c15),
 * and the walk follows the child holding that token, else stops with it as the bonus -- the
 * sequential point-mass rejection scheme (accept child t with probability p(t) / remaining
 * mass), lossless for deterministic top-k children.  Same layouts and preconditions as
 * smart_verify_accept; `seed` selects the random stream (vary it per decode step).
 * SMART_EINVAL if temperature is not > 0. */
smart_status smart_verify_sample(smart_ctx* ctx, const void* d_target, int64_t ld, double temperature,
                                 uint64_t seed, int32_t* d_accept_len, int32_t* d_accept_path,
                                 int32_t* d_bonus, void* stream);

/* Convenience: begin + d x (expand, select) + mask + verify for ROWS_NODE pools, enqueued on
 * one stream (graph-capturable).  Same semantics as the individual calls. */
smart_status smart_run_step(smart_ctx* ctx, const int32_t* d_root_tok, const int32_t* d_root_pos,
                            const void* d_draft, int64_t ld, const void* d_target, int64_t ld_t,
                            uint32_t* d_mask, int32_t* d_pos, int32_t* d_parent, int32_t* d_tok,
                            int32_t* d_tree_len, int32_t* d_accept_len, int32_t* d_accept_path,
                            int32_t* d_bonus, void* stream);

/* ---- inspection (synchronising; tests, stats) -------------------------------------------- */

smart_status smart_get_stats(smart_ctx* ctx, smart_stats* out);

/* Host copies of the tree state: n_nodes [batch_local]; tok/parent/depth [batch_local*T]
 * int32; p/cum [batch_local*T] float.  Any pointer may be NULL. */
smart_status smart_get_tree(smart_ctx* ctx, int32_t* n_nodes, int32_t* tok, int32_t* parent,
                            int32_t* depth, float* p, float* cum);

/* Host copy of layer `layer`'s candidates (frontier order, k per row): count [1];
 * ints [n][4] = (local request, parent node, token, c = slot*k + rank);
 * floats [n][3] = (p, cum, benefit b); admitted [n] int32.  cap = capacity in records. */
smart_status smart_get_candidates(smart_ctx* ctx, int32_t layer, int64_t cap, int32_t* count,
                                  int32_t* ints, float* floats, int32_t* admitted);

const char* smart_last_error(const smart_ctx* ctx);
const char* smart_status_string(smart_status s);

#ifdef __cplusplus
}
#endif
#endif /* SMART_H */
