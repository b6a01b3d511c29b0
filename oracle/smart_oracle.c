/*
 * smart_oracle.c — TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * Plain fp64 scalar reference of the SMART hot path, written from the paper
 * (arXiv 2604.09731, PAPER.md) in the order and notation of Algorithm 1
 * (P:849-876).  No blocking, fusion or reordering beyond what the algorithm
 * states; library primitives (exp, pow) only.  Readings where the paper is
 * silent/ambiguous are the Q# items of DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
 * `--impl reference` legs may load this code.  It shares nothing with the
 * CUDA path in paper_2604_09731_b200/csrc.
 *
 * Pins: every function is checked by tests/test_oracle_*.py
 * against paper/SPEC worked values, closed forms, brute force on tiny
 * inputs and invariants.  Nothing here is "parity unpinned" except the cost
 * constants themselves (Q18: the paper never prints its fitted values).
 */
#include "smart_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EXP_CLAMP 700.0 /* S:133, Q17 */

static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n > 0 ? n : 1; }

/* ------------------------------------------------------------------------ */
/* Cost model                                                                */
/* ------------------------------------------------------------------------ */

/* Eq.(4): C_draft(T) = lambda*|T| + beta */
double orc_cost_draft(const orc_cost* c, double x) { return c->lambda * x + c->beta; }

/* Eq.(5): C_verify(T) = gamma*(exp(delta*|T|^rho) - 1) + eta, exponent clamped (Q17) */
double orc_cost_verify(const orc_cost* c, double x, int* sat) {
  double a = c->delta * pow(x, c->rho);
  if (a > EXP_CLAMP) {
    a = EXP_CLAMP;
    if (sat) *sat = 1;
  }
  return c->gamma * (exp(a) - 1.0) + c->eta;
}

/* C_spec = C_draft + C_verify, Eq.(9) */
double orc_cost_spec(const orc_cost* c, double x, int* sat) {
  return orc_cost_draft(c, x) + orc_cost_verify(c, x, sat);
}

/* Marginal cost of one more node at current size N.
 * DERIVATIVE: Eq.(15), evaluated at M = max(N,1) (Q5).
 * DIFFERENCE: cost(N+1) - cost(N), the Delta n = 1 increment Eq.(14) approximates. */
double orc_dc(const orc_cost* c, int marginal, int64_t N, int* sat) {
  if (marginal == ORC_DIFFERENCE) {
    return orc_cost_spec(c, (double)(N + 1), sat) - orc_cost_spec(c, (double)N, sat);
  }
  double M = (double)(N < 1 ? 1 : N);
  double a = c->delta * pow(M, c->rho);
  if (a > EXP_CLAMP) {
    a = EXP_CLAMP;
    if (sat) *sat = 1;
  }
  return c->lambda + c->gamma * c->delta * c->rho * pow(M, c->rho - 1.0) * exp(a);
}

/* Batch speedup S(E,N) = c_T*(omega*b + E) / (b*cost(N)) (Eq.(1) generalised; Q4, Q13, Q19).
 * 0/0 := 0. */
double orc_speedup(const orc_cost* c, int omega, int b, double E, int64_t N) {
  double C = orc_cost_spec(c, (double)N, NULL);
  double num = c->c_T * ((double)omega * (double)b + E);
  if (C <= 0.0) return 0.0;
  return num / ((double)b * C);
}

/* Eq.(12)/(16): alpha * dT/dS - cT/cS; cS == 0 -> second term 0. */
double orc_delta_j(double alpha, double d_target, double d_spec, double c_target, double c_spec) {
  double g = (c_spec > 0.0) ? c_target / c_spec : 0.0;
  return alpha * d_target / d_spec - g;
}

/* ------------------------------------------------------------------------ */
/* Acceptance models                                                         */
/* ------------------------------------------------------------------------ */

/* Eq.(2): L^tree = (1/|P|) sum_{paths} sum_{j} P(x_{1:j}); root-only tree -> 0
 * (S:212).  Node 0 is the root; parent[i] < i.  Plain definition: for every leaf, walk to
 * the root summing cum over the drafted nodes on the way. */
double orc_l_tree_path_mean(int32_t n, const int32_t* parent, const double* cum) {
  int32_t i, j;
  double total = 0.0;
  int32_t leaves = 0;
  for (i = 0; i < n; i++) {
    int is_leaf = 1;
    for (j = i + 1; j < n; j++)
      if (parent[j] == i) { is_leaf = 0; break; }
    if (!is_leaf) continue;
    leaves++;
    for (j = i; j != 0; j = parent[j]) total += cum[j];
  }
  return leaves ? total / (double)leaves : 0.0;
}

/* P:160 "expected number of consecutively accepted tokens equals the sum of the
 * probabilities that each prefix is accepted": E = sum over drafted nodes of cum (Q11). */
double orc_l_tree_node_sum(int32_t n, const double* cum) {
  double s = 0.0;
  int32_t i;
  for (i = 1; i < n; i++) s += cum[i];
  return s;
}

/* ------------------------------------------------------------------------ */
/* A1: softmax + top-k of one row                                            */
/* ------------------------------------------------------------------------ */

static double logit_at(const void* row, int dtype, int64_t v) {
  if (dtype == ORC_BF16) {
    uint16_t h = ((const uint16_t*)row)[v];
    uint32_t bits = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &bits, 4);
    return (double)f;
  }
  return (double)((const float*)row)[v];
}

/* "better" in the top-k / ranking order: larger value, then lower index (Q9) */
static int better_xi(double xa, int64_t ia, double xb, int64_t ib) {
  if (xa > xb) return 1;
  if (xa < xb) return 0;
  return ia < ib;
}

int orc_topk_softmax(const void* row, int dtype, int V, int k,
                     int32_t* tok, double* p, double* m_out, double* Z_out) {
  int64_t v;
  double m = -INFINITY, Z = 0.0;
  int j, i;
  for (v = 0; v < V; v++) {
    double x = logit_at(row, dtype, v);
    if (isnan(x) || x == INFINITY) return 2; /* Q23 */
    if (x > m) m = x;
  }
  if (m == -INFINITY) return 2; /* all -inf: softmax undefined (Q23) */
  for (v = 0; v < V; v++) Z += exp(logit_at(row, dtype, v) - m); /* index order */
  /* top-k: pick the best remaining element k times (plain definition of a stable
   * descending sort's first k entries). */
  /* (the j-th entry is the best element ranked strictly after entry j-1) */
  double px = 0.0;
  int64_t pi = -1;
  (void)i;
  for (j = 0; j < k; j++) {
    int64_t best = -1;
    double bx = 0.0;
    for (v = 0; v < V; v++) {
      double x = logit_at(row, dtype, v);
      if (j > 0 && !better_xi(px, pi, x, v)) continue; /* already ranked */
      if (best < 0 || better_xi(x, v, bx, best)) { best = v; bx = x; }
    }
    tok[j] = (int32_t)best;
    p[j] = exp(bx - m) / Z; /* draft probability at tau = 1 (Q10) */
    px = bx;
    pi = best;
  }
  if (m_out) *m_out = m;
  if (Z_out) *Z_out = Z;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* One decode step: Algorithm 1 over a batch + A7 + A8           */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t r;      /* global request */
  int32_t parent; /* parent node index within request r */
  int32_t tok;
  int32_t c;      /* slot(parent)*k + rank: canonical candidate index (Q20) */
  double p, cum, b;
  int32_t admitted;
} cand_t;

/* order used by A3 (within a request): b desc, c asc */
static int before_req(const cand_t* a, const cand_t* b) {
  if (a->b > b->b) return 1;
  if (a->b < b->b) return 0;
  return a->c < b->c;
}
/* order used by A4 (batch-global): b desc, r asc, c asc (Q9) */
static int before_glob(const cand_t* a, const cand_t* b) {
  if (a->b > b->b) return 1;
  if (a->b < b->b) return 0;
  if (a->r != b->r) return a->r < b->r;
  return a->c < b->c;
}

/* plain insertion sort on an array of pointers */
static void sort_ptrs(cand_t** v, int64_t n, int (*before)(const cand_t*, const cand_t*)) {
  int64_t i, j;
  for (i = 1; i < n; i++) {
    cand_t* x = v[i];
    for (j = i; j > 0 && before(x, v[j - 1]); j--) v[j] = v[j - 1];
    v[j] = x;
  }
}

static double rel_gap(double a, double b) {
  double s = fabs(a) > fabs(b) ? fabs(a) : fabs(b);
  if (s == 0.0) return INFINITY;
  return fabs(a - b) / s;
}

int orc_step(const orc_config* cfg, const orc_cost* cost,
             const void* draft, int64_t ld, int64_t layer_stride,
             const void* target, int64_t ld_t,
             const int32_t* root_tok, const int32_t* root_pos,
             int32_t* n_nodes, int32_t* tok, int32_t* parent, int32_t* depth, int32_t* pos,
             double* p, double* cum, uint32_t* mask,
             int32_t* accept_len, int32_t* accept_path, int32_t* bonus,
             double* trace, int64_t capc, int32_t* cand_i, double* cand_d, double* summary) {
  const int b = cfg->b, k = cfg->k, d = cfg->d, T = cfg->T, V = cfg->V;
  const int64_t Wq = cfg->W > 0 ? cfg->W : (int64_t)1 << 40; /* W = 0: unlimited (Q12) */
  const int esz = cfg->dtype == ORC_BF16 ? 2 : 4;
  const int MW = (T + 31) / 32;
  int64_t B, r, i, j, l;
  int rc = 0, sat_any = 0, first_amb = 0, layers_exec = 0;

  if (b < 1 || k < 1 || k > V || d < 0 || T < 1 || cfg->alpha <= 0.0 || cfg->alpha > 1.0) return 1;
  /* Alg.1 line 1, floor (Q2); b_budget > b: this batch is one replica's share of the
   * b_budget requests the budget is split over (cost_scope LOCAL, Q34) */
  B = cfg->B_verify / (cfg->b_budget > 0 ? cfg->b_budget : b);
  if (B < 1) return 1;

  /* per-request state: S_0 = {root}, A_0 = {root} */
  int32_t* n = calloc(b, sizeof(int32_t));            /* drafted nodes n_r (root excluded, Q1) */
  double* E = calloc(b, sizeof(double));              /* E_r: acceptance estimate of tree r    */
  int32_t* act = malloc(sizeof(int32_t) * b * T);     /* A_r: node indices, canonical order   */
  int32_t* nact = calloc(b, sizeof(int32_t));
  int32_t* nact_next = calloc(b, sizeof(int32_t));
  int32_t* act_next = malloc(sizeof(int32_t) * b * T);
  int32_t* topi = malloc(sizeof(int32_t) * k * ((int64_t)b * T + 1)); /* per frontier row */
  double* topp = malloc(sizeof(double) * k * ((int64_t)b * T + 1));
  const char** rowp = malloc(sizeof(char*) * ((int64_t)b * T + 1));
  int* rowrc = malloc(sizeof(int) * ((int64_t)b * T + 1));
  int64_t cap = (int64_t)b * T * k + 1;
  cand_t* cand = malloc(sizeof(cand_t) * cap);
  cand_t** ord = malloc(sizeof(cand_t*) * cap);
  cand_t** elig = malloc(sizeof(cand_t*) * cap);
  int64_t* kid = calloc((size_t)b * T, sizeof(int64_t)); /* k-ary index (ROWS_KARY only) */

  for (r = 0; r < b; r++) {
    n_nodes[r] = 1;
    tok[r * T] = root_tok ? root_tok[r] : -1;
    parent[r * T] = -1;
    depth[r * T] = 0;
    p[r * T] = 1.0;   /* root: p = cum = 1 */
    cum[r * T] = 1.0;
    act[r * T] = 0;
    nact[r] = 1;
  }
  memset(trace, 0, sizeof(double) * (size_t)(d > 0 ? d : 1) * ORC_TRACE_F);

  for (l = 1; l <= d; l++) { /* Alg.1 line 3 */
    double* tr = trace + (l - 1) * ORC_TRACE_F;
    int64_t nc = 0, rows = 0, frow = 0;
    int sat = 0;
    /* ---- A1/A2: U_l(A_{l-1}) — top-k candidates of every frontier node ----
     * (rows are independent: their softmax/top-k may run on several threads, orc_set_threads) */
    for (r = 0; r < b; r++) {
      for (i = 0; i < nact[r]; i++) {
        int32_t u = act[r * T + i];
        const char* row;
        if (cfg->row_mode == ORC_ROWS_NODE)
          row = (const char*)draft + ((int64_t)r * T + u) * ld * esz;
        else if (cfg->row_mode == ORC_ROWS_KARY) /* path-keyed: full k-ary tree index */
          row = (const char*)draft + ((int64_t)r * layer_stride + kid[r * T + u]) * ld * esz;
        else if (cfg->row_mode == ORC_ROWS_POSITION) /* DFLASH: position l's row for every node */
          row = (const char*)draft + ((int64_t)r * layer_stride + (l - 1)) * ld * esz;
        else
          row = (const char*)draft + ((l - 1) * layer_stride + frow * ld) * esz;
        rowp[frow] = row;
        frow++;
      }
    }
    {
      int64_t q;
#pragma omp parallel for num_threads(g_threads) schedule(dynamic, 1) if (g_threads > 1)
      for (q = 0; q < frow; q++)
        rowrc[q] = orc_topk_softmax(rowp[q], cfg->dtype, V, k, topi + q * k, topp + q * k, NULL, NULL);
      for (q = 0; q < frow; q++)
        if (rowrc[q]) { rc = rowrc[q]; goto done; }
    }
    frow = 0;
    for (r = 0; r < b; r++) {
      for (i = 0; i < nact[r]; i++) {
        int32_t u = act[r * T + i];
        for (j = 0; j < k; j++) {
          cand_t* c = &cand[nc++];
          c->r = (int32_t)r;
          c->parent = u;
          c->tok = topi[frow * k + j];
          c->c = (int32_t)(i * k + j);
          c->p = topp[frow * k + j];
          c->cum = cum[r * T + u] * topp[frow * k + j]; /* Eq.(3): cum(parent) * p */
          c->admitted = 0;
        }
        frow++;
        rows++;
      }
    }
    if (rows == 0) break; /* A_{l-1} empty everywhere */
    layers_exec++;
    tr[0] = (double)rows;
    tr[1] = (double)nc;
    tr[12] = 1.0;

    /* ---- A3: marginal benefit b_u = cum/|P_r| (Eq.(13); |P| frozen at layer
     *      start, Q6) or cum (NODE_SUM); per-request eligibility min(B - n_r, W) (Q3, Q12) ---- */
    double min_margin = INFINITY;
    int64_t ne = 0, s0 = 0;
    for (r = 0; r < b; r++) {
      double D = 1.0;
      if (cfg->accept_model == ORC_PATH_MEAN) {
        int32_t leaves = 0;
        for (i = 0; i < n_nodes[r]; i++) {
          int is_leaf = 1;
          for (j = i + 1; j < n_nodes[r]; j++)
            if (parent[r * T + j] == i) { is_leaf = 0; break; }
          leaves += is_leaf;
        }
        D = (double)leaves; /* |P_r| = number of root-to-leaf paths */
      }
      int64_t m = 0;
      while (s0 + m < nc && cand[s0 + m].r == r) {
        cand[s0 + m].b = cand[s0 + m].cum / D;
        ord[m] = &cand[s0 + m];
        m++;
      }
      sort_ptrs(ord, m, before_req);
      int64_t q = B - n[r];
      if (q > Wq) q = Wq;
      if (q < 0) q = 0;
      for (i = 0; i < m && i < q; i++) elig[ne++] = ord[i];
      if (q > 0 && q < m && ord[q - 1]->b != ord[q]->b) {
        double g = rel_gap(ord[q - 1]->b, ord[q]->b);
        if (g < min_margin) min_margin = g;
      }
      s0 += m;
    }
    tr[2] = (double)ne;

    /* ---- A4: batch-global ranking (b desc, r asc, c asc) ---- */
    sort_ptrs(elig, ne, before_glob);

    /* ---- A5: global terms on S_{l-1} (Alg.1 lines 5-6) and the decision rule
     *      Eq.(16) — FROZEN: each candidate against the frozen state; PREFIX: sequentially,
     *      stop at the first rejection (Q7).  Decisions compare alpha*c_T*b/dc against
     *      c_T*(omega*b+E)/cost(N) (= b * S; the 1/b of S cancels on both sides). ---- */
    int64_t N0 = 0;
    double E0 = 0.0;
    for (r = 0; r < b; r++) { N0 += n[r]; E0 += E[r]; } /* global request order */
    double C0 = orc_cost_spec(cost, (double)N0, &sat);
    double dc0 = orc_dc(cost, cfg->marginal, N0, &sat);
    double Sb0 = C0 > 0.0 ? cost->c_T * ((double)cfg->omega * b + E0) / C0 : 0.0;
    tr[4] = (double)N0;
    tr[5] = E0;
    tr[6] = Sb0 / b;
    tr[9] = dc0;
    int64_t jstar = 0;
    double Eacc = E0;
    double bestS = Sb0;
    int64_t bestj = 0;
    if (cfg->selection == ORC_FROZEN) {
      for (j = 0; j < ne; j++) {
        double lhs = cfg->alpha * cost->c_T * elig[j]->b / dc0;
        double g = rel_gap(lhs, Sb0);
        if (g < min_margin) min_margin = g;
        if (lhs > Sb0) { elig[j]->admitted = 1; jstar++; } /* strict ">" (Q8) */
      }
      /* with b sorted descending the admitted set is a prefix; count it */
    } else {
      for (j = 0; j < ne; j++) {
        int64_t Nj = N0 + j;
        double Cj = orc_cost_spec(cost, (double)Nj, &sat);
        double Sbj = Cj > 0.0 ? cost->c_T * ((double)cfg->omega * b + Eacc) / Cj : 0.0;
        double dcj = orc_dc(cost, cfg->marginal, Nj, &sat);
        double lhs = cfg->alpha * cost->c_T * elig[j]->b / dcj;
        double g = rel_gap(lhs, Sbj);
        if (g < min_margin) min_margin = g;
        if (!(lhs > Sbj)) break; /* no skipping */
        elig[j]->admitted = 1;
        jstar++;
        Eacc += elig[j]->b;
      }
    }
    /* cut gap: if the last admitted and the first rejected swap, the set changes */
    if (jstar > 0 && jstar < ne && elig[jstar - 1]->b != elig[jstar]->b) {
      double g = rel_gap(elig[jstar - 1]->b, elig[jstar]->b);
      if (g < min_margin) min_margin = g;
    }
    /* report argmax_j S_j over prefixes j = 0..|L| (smallest j on ties) */
    {
      double Ej = E0;
      for (j = 1; j <= ne; j++) {
        Ej += elig[j - 1]->b;
        double Cj = orc_cost_spec(cost, (double)(N0 + j), &sat);
        double Sbj = Cj > 0.0 ? cost->c_T * ((double)cfg->omega * b + Ej) / Cj : 0.0;
        if (Sbj > bestS) { bestS = Sbj; bestj = j; }
      }
    }
    tr[3] = (double)jstar;
    tr[8] = (double)bestj;
    tr[10] = min_margin;
    tr[11] = min_margin < cfg->margin_eps ? 1.0 : 0.0;
    tr[13] = sat ? 1.0 : 0.0;
    if (sat) sat_any = 1;
    if (tr[11] != 0.0 && first_amb == 0) first_amb = (int)l;

    /* ---- A6: commit A_l in canonical order (c asc) — Eq.(7) S_l = S_{l-1} ∪ A_l ---- */
    s0 = 0;
    for (r = 0; r < b; r++) {
      int64_t m = 0;
      while (s0 + m < nc && cand[s0 + m].r == r) m++;
      nact_next[r] = 0;
      for (i = 0; i < m; i++) { /* cand of r are stored in c order already */
        cand_t* c = &cand[s0 + i];
        if (!c->admitted) continue;
        int32_t node = n_nodes[r];
        tok[r * T + node] = c->tok;
        parent[r * T + node] = c->parent;
        depth[r * T + node] = (int32_t)l;
        p[r * T + node] = c->p;
        cum[r * T + node] = c->cum;
        kid[r * T + node] = kid[r * T + c->parent] * k + (c->c % k) + 1;
        n_nodes[r]++;
        n[r]++;
        act_next[r * T + nact_next[r]++] = node;
      }
      /* E_r on the committed tree */
      if (cfg->accept_model == ORC_PATH_MEAN)
        E[r] = orc_l_tree_path_mean(n_nodes[r], parent + r * T, cum + r * T);
      else
        E[r] = orc_l_tree_node_sum(n_nodes[r], cum + r * T);
      /* A_l becomes the next frontier unless the request is finished:
       * A_l empty or |S_l| >= B (Alg.1 line 10) */
      if (n[r] >= B) nact_next[r] = 0;
      s0 += m;
    }
    {
      double Ea = 0.0;
      int64_t Na = 0;
      for (r = 0; r < b; r++) { Ea += E[r]; Na += n[r]; }
      tr[7] = orc_speedup(cost, cfg->omega, b, Ea, Na);
    }
    /* candidate dump (for score parity) */
    if (cand_i && cand_d) {
      for (i = 0; i < nc && i < capc; i++) {
        int32_t* ci = cand_i + ((l - 1) * capc + i) * 5;
        double* cd = cand_d + ((l - 1) * capc + i) * 3;
        ci[0] = cand[i].r; ci[1] = cand[i].parent; ci[2] = cand[i].tok; ci[3] = cand[i].c;
        ci[4] = cand[i].admitted;
        cd[0] = cand[i].p; cd[1] = cand[i].cum; cd[2] = cand[i].b;
      }
    }
    for (r = 0; r < b; r++) {
      nact[r] = nact_next[r];
      for (i = 0; i < nact[r]; i++) act[r * T + i] = act_next[r * T + i];
    }
  }

  /* ---- A7: ancestor-or-self mask, position ids (Q20, Q21) ---- */
  for (r = 0; r < b; r++) {
    for (i = 0; i < T; i++) {
      uint32_t* row = mask + ((int64_t)r * T + i) * MW;
      for (j = 0; j < MW; j++) row[j] = 0;
      if (i >= n_nodes[r]) {
        pos[r * T + i] = 0;
        if (i > 0) { tok[r * T + i] = -1; parent[r * T + i] = -1; depth[r * T + i] = 0; }
        continue;
      }
      for (j = i; j >= 0; j = parent[r * T + j]) row[j / 32] |= 1u << (j % 32);
      pos[r * T + i] = (root_pos ? root_pos[r] : 0) + depth[r * T + i];
    }
  }

  /* ---- A8: greedy (T=0) tree verification walk (Q16); requests are independent ---- */
  int64_t sum_a = 0, sum_n = 0;
  int nan_seen = 0;
  for (r = 0; r < b; r++) sum_n += n[r];
#pragma omp parallel for num_threads(g_threads) schedule(dynamic, 1) reduction(+ : sum_a) reduction(| : nan_seen) if (g_threads > 1)
  for (r = 0; r < b; r++) {
    int64_t jj;
    accept_len[r] = 0;
    for (jj = 0; jj < d; jj++) accept_path[r * d + jj] = -1;
    bonus[r] = -1;
    if (!target) continue;
    int32_t cur = 0;
    for (;;) {
      const char* row = (const char*)target + ((int64_t)r * T + cur) * ld_t * esz;
      int64_t best = -1;
      double bx = 0.0;
      int bad = 0;
      for (jj = 0; jj < V; jj++) {
        double x = logit_at(row, cfg->dtype, jj);
        if (isnan(x)) { bad = 1; break; }
        if (best < 0 || better_xi(x, jj, bx, best)) { best = jj; bx = x; }
      }
      if (bad) { nan_seen = 1; break; }
      int32_t next = -1;
      for (jj = cur + 1; jj < n_nodes[r]; jj++)
        if (parent[r * T + jj] == cur && tok[r * T + jj] == best) { next = (int32_t)jj; break; }
      if (next < 0) { bonus[r] = (int32_t)best; break; }
      accept_path[r * d + accept_len[r]] = next;
      accept_len[r]++;
      cur = next;
    }
    sum_a += accept_len[r];
  }
  if (nan_seen) { rc = 2; goto done; }

  {
    double Ea = 0.0;
    int64_t Na = 0;
    for (r = 0; r < b; r++) {
      /* final E recomputed from scratch on the final tree (closed-form pin) */
      if (cfg->accept_model == ORC_PATH_MEAN)
        Ea += orc_l_tree_path_mean(n_nodes[r], parent + r * T, cum + r * T);
      else
        Ea += orc_l_tree_node_sum(n_nodes[r], cum + r * T);
      Na += n[r];
    }
    summary[0] = Ea;
    summary[1] = (double)Na;
    summary[2] = orc_speedup(cost, cfg->omega, b, Ea, Na);
    summary[3] = (double)sum_a;
    summary[4] = sum_n ? (double)sum_a / (double)sum_n : 0.0; /* beta */
    summary[5] = (double)first_amb;
    summary[6] = (double)layers_exec;
    summary[7] = (double)sat_any;
    summary[8] = (double)B;
  }

done:
  free(n); free(E); free(act); free(nact); free(nact_next); free(act_next);
  free(topi); free(topp); free(rowp); free(rowrc); free(cand); free(ord); free(elig); free(kid);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* NEXT #1: tree verification at temperature tau > 0 (Q31)                   */
/* ------------------------------------------------------------------------ */

static uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}

/* counter-based generator: a per-(request, node) 32-bit row key from SplitMix64, then per token
 * v the lowbias32 integer hash of rowkey + v * 0x9e3779b9 (all arithmetic mod 2^32 / 2^64) */
static uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

uint64_t orc_hash(uint64_t seed, int64_t r, int64_t u, int64_t v) {
  const uint64_t rk = mix64(seed + (((uint64_t)r << 22) | (uint64_t)u) * 0x9e3779b97f4a7c15ULL);
  return lowbias32((uint32_t)(rk >> 32) + (uint32_t)v * 0x9e3779b9U);
}

/* 23-bit uniform in (0, 1): (h >> 9) + 1/2 over 2^23 (exact in fp32 as well) */
double orc_uniform(uint64_t seed, int64_t r, int64_t u, int64_t v) {
  return ((double)(orc_hash(seed, r, u, v) >> 9) + 0.5) / 8388608.0;
}

int orc_verify_sample(int dtype, int V, int T, int b, int r_off, int d, const void* target, int64_t ld_t,
                      const int32_t* n_nodes, const int32_t* parent, const int32_t* tok, double tau,
                      uint64_t seed, int32_t* accept_len, int32_t* accept_path, int32_t* bonus,
                      double* margin) {
  if (!(tau > 0.0) || V < 1 || T < 1 || b < 0 || d < 0 || !target) return 1;
  const int esz = dtype == ORC_BF16 ? 2 : 4;
  const int D = d > 0 ? d : 1;
  for (int r = 0; r < b; r++) {
    const int64_t rg = (int64_t)r_off + r;
    accept_len[r] = 0;
    for (int i = 0; i < D; i++) accept_path[r * D + i] = -1;
    bonus[r] = -1;
    double mg = INFINITY;
    int32_t cur = 0;
    for (;;) {
      /* one sample from softmax(logits/tau) at node cur: Gumbel-max */
      const char* row = (const char*)target + ((int64_t)r * T + cur) * ld_t * esz;
      int64_t best = -1;
      double by = 0.0, second = -INFINITY;
      for (int64_t v = 0; v < V; v++) {
        const double x = logit_at(row, dtype, v);
        if (isnan(x)) return 2;
        const double U = orc_uniform(seed, rg, cur, v);
        const double y = x / tau - log(-log(U));
        if (best < 0 || y > by) {  /* ties keep the lower token id */
          if (best >= 0) second = by;
          best = v;
          by = y;
        } else if (y > second) {
          second = y;
        }
      }
      if (by - second < mg) mg = by - second;
      int32_t next = -1;
      for (int32_t j = cur + 1; j < n_nodes[r]; j++)
        if (parent[r * T + j] == cur && tok[r * T + j] == best) { next = j; break; }
      if (next < 0) { bonus[r] = (int32_t)best; break; }
      if (accept_len[r] < D) accept_path[r * D + accept_len[r]] = next;
      accept_len[r]++;
      cur = next;
    }
    if (margin) margin[r] = mg;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT #3: the likelihood-maximising two-stage baseline (Q32)               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t layer, c, parent_e, tok, exp_node; /* exp_node: expanded-tree index, -1 if not expanded */
  double p, cum;
} bcand_t;

/* rerank order: cum desc, layer asc, c asc */
static int before_rerank(const bcand_t* a, const bcand_t* b) {
  if (a->cum > b->cum) return 1;
  if (a->cum < b->cum) return 0;
  if (a->layer != b->layer) return a->layer < b->layer;
  return a->c < b->c;
}

int orc_baseline_step(const orc_config* cfg, const void* draft, int64_t ld, const void* target, int64_t ld_t,
                      const int32_t* root_tok, const int32_t* root_pos, int32_t* n_nodes, int32_t* tok,
                      int32_t* parent, int32_t* depth, int32_t* pos, double* p, double* cum, uint32_t* mask,
                      int32_t* accept_len, int32_t* accept_path, int32_t* bonus, int32_t* n_exp) {
  const int b = cfg->b, k = cfg->k, d = cfg->d, T = cfg->T, V = cfg->V, w = cfg->W;
  const int esz = cfg->dtype == ORC_BF16 ? 2 : 4;
  const int MW = (T + 31) / 32;
  const int D = d > 0 ? d : 1;
  if (b < 1 || k < 1 || k > V || d < 0 || T < 1 || w < 1) return 1;
  const int64_t g = cfg->B_verify / b;
  if (g < 1 || T < 1 + g) return 1;
  const int64_t cap = (int64_t)(d > 0 ? d : 1) * w * k + 1;
  bcand_t* all = malloc(sizeof(bcand_t) * cap);
  bcand_t** ord = malloc(sizeof(bcand_t*) * cap);
  int32_t* topi = malloc(sizeof(int32_t) * k);
  double* topp = malloc(sizeof(double) * k);
  /* expanded tree (per request): cum and the candidate it came from */
  const int64_t te = 1 + (int64_t)w * (d > 0 ? d : 1);
  double* ecum = malloc(sizeof(double) * te);
  int32_t* efront = malloc(sizeof(int32_t) * te);
  int32_t* newidx = malloc(sizeof(int32_t) * te);
  int rc = 0;
  for (int r = 0; r < b; r++) {
    int64_t na = 0;
    int32_t ne = 1, nf = 1;
    ecum[0] = 1.0;
    efront[0] = 0;
    for (int l = 1; l <= d && nf > 0; l++) {
      const int64_t l0 = na;
      for (int i = 0; i < nf; i++) {
        const int32_t u = efront[i];
        const char* row = cfg->row_mode == ORC_ROWS_POSITION /* DFLASH position rows */
                              ? (const char*)draft + ((int64_t)r * d + (l - 1)) * ld * esz
                              : (const char*)draft + ((int64_t)r * T + u) * ld * esz;
        rc = orc_topk_softmax(row, cfg->dtype, V, k, topi, topp, NULL, NULL);
        if (rc) goto done;
        for (int j = 0; j < k; j++) {
          bcand_t* c = &all[na++];
          c->layer = l;
          c->c = i * k + j;
          c->parent_e = u;
          c->tok = topi[j];
          c->p = topp[j];
          c->cum = ecum[u] * topp[j]; /* Eq.(3) */
          c->exp_node = -1;
        }
      }
      /* the layer's top-w by (cum desc, c asc) are expanded next */
      const int64_t nl = na - l0;
      for (int64_t q = 0; q < nl; q++) ord[q] = &all[l0 + q];
      for (int64_t x = 1; x < nl; x++) { /* insertion sort: cum desc, c asc */
        bcand_t* y = ord[x];
        int64_t z;
        for (z = x; z > 0 && (y->cum > ord[z - 1]->cum || (y->cum == ord[z - 1]->cum && y->c < ord[z - 1]->c)); z--)
          ord[z] = ord[z - 1];
        ord[z] = y;
      }
      const int64_t take = nl < w ? nl : w;
      /* commit in canonical (c asc) order */
      nf = 0;
      for (int64_t q = 0; q < nl; q++) {
        bcand_t* c = &all[l0 + q];
        int sel = 0;
        for (int64_t z = 0; z < take; z++) sel |= (ord[z] == c);
        if (!sel) continue;
        c->exp_node = ne;
        ecum[ne] = c->cum;
        efront[nf++] = ne;
        ne++;
      }
    }
    n_exp[r] = ne;
    /* rerank: top-g of all generated candidates */
    for (int64_t q = 0; q < na; q++) ord[q] = &all[q];
    for (int64_t x = 1; x < na; x++) {
      bcand_t* y = ord[x];
      int64_t z;
      for (z = x; z > 0 && before_rerank(y, ord[z - 1]); z--) ord[z] = ord[z - 1];
      ord[z] = y;
    }
    const int64_t keep = na < g ? na : g;
    /* final numbering in (layer, c) order = the order of `all` */
    for (int64_t e = 0; e < te; e++) newidx[e] = -1;
    newidx[0] = 0;
    int32_t nn = 1;
    const int64_t o = (int64_t)r * T;
    tok[o] = root_tok ? root_tok[r] : -1;
    parent[o] = -1;
    depth[o] = 0;
    p[o] = 1.0;
    cum[o] = 1.0;
    for (int64_t q = 0; q < na; q++) {
      bcand_t* c = &all[q];
      int kept = 0;
      for (int64_t z = 0; z < keep; z++) kept |= (ord[z] == c);
      if (!kept) continue;
      if (newidx[c->parent_e] < 0) { rc = 1; goto done; } /* closure violated (cannot happen) */
      tok[o + nn] = c->tok;
      parent[o + nn] = newidx[c->parent_e];
      depth[o + nn] = c->layer;
      p[o + nn] = c->p;
      cum[o + nn] = c->cum;
      if (c->exp_node >= 0) newidx[c->exp_node] = nn;
      nn++;
    }
    n_nodes[r] = nn;
    /* A7: mask rows and positions (padding rows zero) */
    for (int32_t i = 0; i < T; i++) {
      uint32_t* mrow = mask + (o + i) * MW;
      for (int ww = 0; ww < MW; ww++) mrow[ww] = 0u;
      if (i >= nn) {
        pos[o + i] = 0;
        if (i > 0) { tok[o + i] = -1; parent[o + i] = -1; depth[o + i] = 0; }
        continue;
      }
      for (int32_t j = i; j >= 0; j = parent[o + j]) mrow[j / 32] |= 1u << (j % 32);
      pos[o + i] = (root_pos ? root_pos[r] : 0) + depth[o + i];
    }
    /* A8: greedy walk */
    accept_len[r] = 0;
    for (int i = 0; i < D; i++) accept_path[r * D + i] = -1;
    bonus[r] = -1;
    if (!target) continue;
    int32_t cur = 0;
    for (;;) {
      const char* row = (const char*)target + (o + cur) * ld_t * esz;
      int64_t best = -1;
      double bx = 0.0;
      for (int64_t v = 0; v < V; v++) {
        const double x = logit_at(row, cfg->dtype, v);
        if (isnan(x)) { rc = 2; goto done; }
        if (best < 0 || better_xi(x, v, bx, best)) { best = v; bx = x; }
      }
      int32_t next = -1;
      for (int32_t j = cur + 1; j < nn; j++)
        if (parent[o + j] == cur && tok[o + j] == best) { next = j; break; }
      if (next < 0) { bonus[r] = (int32_t)best; break; }
      if (accept_len[r] < D) accept_path[r * D + accept_len[r]] = next;
      accept_len[r]++;
      cur = next;
    }
  }
done:
  free(all); free(ord); free(topi); free(topp); free(ecum); free(efront); free(newidx);
  return rc;
}
