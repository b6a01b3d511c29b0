/*
 * smart_oracle.h — TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * Plain, slow, obviously-correct fp64 CPU reference of the SMART hot path
 * (arXiv 2604.09731, "SMART: When is it Actually Worth Expanding a Speculative
 * Tree?").  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load liboracle.so.  It shares no code, header,
 * table or helper with paper_2604_09731_b200/csrc (the CUDA path) and neither
 * side includes or imports the other.
 *
 * Citation keys: P:n = line n of PAPER.md (the paper), S:n = line n of SPEC.md,
 * Q# = a reading listed in DESIGN.md §3 (taken from SURVEY.md §8(c)).
 *
 * Parity pins: see oracle/README and DESIGN.md §4.  Every function below is
 * pinned by at least one `-m "not gpu"` test in tests/test_oracle_*.py.
 */
#ifndef SMART_ORACLE_H
#define SMART_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Cost-model constants: Eq.(4) lambda,beta; Eq.(5) gamma,delta,rho,eta; Eq.(1) c_T. */
typedef struct {
  double lambda, beta, gamma, delta, rho, eta, c_T;
} orc_cost;

enum { ORC_PREFIX = 0, ORC_FROZEN = 1 };       /* Q7  */
enum { ORC_NODE_SUM = 0, ORC_PATH_MEAN = 1 };  /* Q11 */
enum { ORC_DERIVATIVE = 0, ORC_DIFFERENCE = 1 };/* Q5  */
enum { ORC_BF16 = 0, ORC_FP32 = 1 };
enum { ORC_ROWS_NODE = 0, ORC_ROWS_FRONTIER = 1, ORC_ROWS_KARY = 2, ORC_ROWS_POSITION = 3 };

typedef struct {
  int32_t V, k, d, W;          /* vocab, top-k, depth, frontier cap (0 = unlimited) */
  int32_t b;                   /* batch size (global)                                */
  int32_t B_verify;            /* total verification budget; B = floor(B_verify/b)  */
  double alpha;                /* discount factor, (0,1]                            */
  int32_t omega;               /* bonus-token term in S (Q19), 0 or 1               */
  int32_t selection, accept_model, marginal, dtype, row_mode;
  int32_t T;                   /* per-request node capacity incl. root (pool rows)  */
  double margin_eps;           /* relative margin below which a decision is flagged (Q24) */
  int32_t b_budget;            /* requests sharing B_verify (the global batch, Q2): B =
                                  floor(B_verify / b_budget); 0 = b.  With b_budget > b the
                                  b requests are one replica's share, costed as their own
                                  batch (cost_scope LOCAL, Q13 / DESIGN.md Q34)              */
} orc_config;

/* worker threads of the row-parallel parts (A1 softmax/top-k rows, A8 target argmax rows);
 * 1 = serial (default).  Only the bench's all-cores baseline raises it. */
void orc_set_threads(int n);

/* ---- closed-form pieces (each pinned separately) ------------------------- */
double orc_cost_draft(const orc_cost* c, double x);             /* Eq.(4) */
double orc_cost_verify(const orc_cost* c, double x, int* sat);  /* Eq.(5), clamp Q17 */
double orc_cost_spec(const orc_cost* c, double x, int* sat);         /* Eq.(4)+(5) */
double orc_dc(const orc_cost* c, int marginal, int64_t N, int* sat); /* Eq.(15) / Q5 */
/* batch speedup, Eq.(1) generalised (Q4,Q13,Q19): c_T*(omega*b+E)/(b*cost(N)), 0/0:=0 */
double orc_speedup(const orc_cost* c, int omega, int b, double E, int64_t N);
/* Eq.(12)/(16): delta_j = alpha*dT/dS - cT/cS (second term 0 when cS==0) */
double orc_delta_j(double alpha, double d_target, double d_spec, double c_target, double c_spec);
/* Eq.(2): expected acceptance length of one tree (path mean), root-only -> 0 */
double orc_l_tree_path_mean(int32_t n, const int32_t* parent, const double* cum);
/* node-sum acceptance model (P:160 prefix argument; Q11) */
double orc_l_tree_node_sum(int32_t n, const double* cum);

/* A1: softmax at tau=1 over all V entries (Q10) + top-k by (x desc, token asc) (Q9).
 * returns 0, or 2 if the row holds NaN/+inf (Q23). */
int orc_topk_softmax(const void* row, int dtype, int V, int k,
                     int32_t* tok, double* p, double* m_out, double* Z_out);

/* One whole decode step (Algorithm 1, with the readings Q1-Q24):
 * expand/select per layer, then mask/pos/parent (A7) and greedy verify (A8).
 *
 * draft:  bf16/fp32 logits.  ROWS_NODE:     row (r, node u) at draft + (r*T + u)*ld
 *                            ROWS_FRONTIER: row i of layer l at draft + (l-1)*layer_stride + i*ld
 *                            ROWS_KARY:     row of the node whose path of top-k ranks gives heap
 *                                           index f (root 0, child j of f: f*k+j+1) at
 *                                           draft + (r*layer_stride + f)*ld  (tests only)
 *                            ROWS_POSITION: DFLASH -- one non-autoregressive forward gives
 *                                           independent per-position distributions; every frontier
 *                                           node of request r at layer l expands with position row
 *                                           l: draft + (r*layer_stride + l-1)*ld, layer_stride =
 *                                           position rows per request (>= d).  With selection
 *                                           BASELINE and W >= g this is the paper's Cartesian
 *                                           product pruned to the top-g by cumulative probability.
 * target: NODE layout [b][T][ld_t] or NULL (skip A8).
 * Output arrays are caller-allocated (sizes in oracle.py).  Returns 0 ok,
 * 1 invalid config, 2 invalid logits (NaN/+inf). */
int orc_step(const orc_config* cfg, const orc_cost* cost,
             const void* draft, int64_t ld, int64_t layer_stride,
             const void* target, int64_t ld_t,
             const int32_t* root_tok, const int32_t* root_pos,
             /* tree outputs [b*T] */
             int32_t* n_nodes, int32_t* tok, int32_t* parent, int32_t* depth, int32_t* pos,
             double* p, double* cum, uint32_t* mask,
             /* verify outputs */
             int32_t* accept_len, int32_t* accept_path, int32_t* bonus,
             /* per-layer trace [d * ORC_TRACE_F] */
             double* trace,
             /* candidate dump [d * capc]: ints (r, parent, tok, c, admitted), doubles (p, cum, b) */
             int64_t capc, int32_t* cand_i, double* cand_d,
             /* summary [ORC_SUM_F] */
             double* summary);

/* NEXT #3 (reading Q32): the likelihood-maximising two-stage baseline of EAGLE-3 / MSD
 * (Fig. 2(a)(b)), per request r:
 *  expand: for l = 1..d, every frontier node (layer l-1, canonical order; A_0 = {root}) gets
 *          its top-k children (A1/A2 as orc_step); the top-w candidates of the layer by
 *          (cum desc, c asc) are committed as expanded nodes (node indices in canonical c order)
 *          and form the next frontier (w = cfg->W, the "global top-k nodes"; Fig. 2: w = k = 2);
 *  rerank: all generated candidates are reranked by (cum desc, layer asc, c asc) and the top
 *          g = floor(B_verify / b) kept (cum never increases along a path, so the kept set is
 *          ancestor-closed by construction); the final tree numbers them in (layer, c) order.
 * Draft rows: NODE layout at (r, expanded node).  Outputs: the final tree, its mask/pos (A7)
 * and the greedy walk (A8, target rows at (r, final node)); n_exp[r] = expanded nodes incl.
 * the root.  Returns 0, 1 bad config, 2 invalid logits. */
int orc_baseline_step(const orc_config* cfg, const void* draft, int64_t ld, const void* target, int64_t ld_t,
                      const int32_t* root_tok, const int32_t* root_pos, int32_t* n_nodes, int32_t* tok,
                      int32_t* parent, int32_t* depth, int32_t* pos, double* p, double* cum, uint32_t* mask,
                      int32_t* accept_len, int32_t* accept_path, int32_t* bonus, int32_t* n_exp);

/* NEXT #1 (reading Q31): tree verification at temperature tau > 0.  Walk from the root of each
 * request: at node u draw the target token by Gumbel-max over the target row,
 *   x* = argmax_v ( logit_v / tau + G_v ),  G_v = -log(-log(U_v)),
 *   U_v = ((h >> 9) + 0.5) / 2^23,  h = orc_hash(seed, r_glob, u, v),
 * follow the child of u whose token is x*, else stop with bonus = x*.  This realises the
 * sequential point-mass rejection scheme (accept child t with probability p(t) / remaining mass,
 * zero t on rejection, bonus from the renormalised residual) with one sample
 * per node, hence losslessly: every emitted token is distributed as softmax(logits / tau).
 * target: NODE layout [b][T][ld_t]; r_glob = r_off + r.  margin[r] (optional) = smallest gap
 * between the best and second-best perturbed logit on r's walk (decision margin, Q24 style).
 * Returns 0, 1 bad arguments, 2 NaN logits. */
int orc_verify_sample(int dtype, int V, int T, int b, int r_off, int d, const void* target, int64_t ld_t,
                      const int32_t* n_nodes, const int32_t* parent, const int32_t* tok, double tau,
                      uint64_t seed, int32_t* accept_len, int32_t* accept_path, int32_t* bonus,
                      double* margin);
/* the counter-based generator: row key rk = SplitMix64(seed + (r << 22 | u) * 0x9e3779b97f4a7c15)
 * (r < 2^42, u < 2^22), h = lowbias32((rk >> 32) + v * 0x9e3779b9) (32-bit), and the 23-bit
 * uniform in (0, 1) it defines */
uint64_t orc_hash(uint64_t seed, int64_t r, int64_t u, int64_t v);
double orc_uniform(uint64_t seed, int64_t r, int64_t u, int64_t v);

#define ORC_TRACE_F 14
/* trace fields: 0 n_rows, 1 n_cand, 2 n_elig, 3 n_admit, 4 N0, 5 E0, 6 S0 (per-request S),
 * 7 S_after, 8 argmax_j S_j, 9 dc(N0), 10 min_margin, 11 ambiguous(0/1), 12 executed(0/1),
 * 13 saturated(0/1) */
#define ORC_SUM_F 9
/* summary: 0 E, 1 N, 2 S_final, 3 sum_accept, 4 beta, 5 first_ambiguous_layer (0 = none),
 * 6 layers_executed, 7 saturated, 8 B */

#ifdef __cplusplus
}
#endif
#endif
