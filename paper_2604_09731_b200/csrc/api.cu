// api.cu — host side of the libsmart C-ABI (include/smart.h): validation, workspace,
// launch sequencing, NCCL exchange for sharded batches, inspection.
//
// No torch, no oracle: this file links only the CUDA runtime (and dlopen()s libnccl.so.2 when
// a context is attached to a multi-rank communicator).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "stream.cuh"

using namespace smart;

bool smart::pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SMART_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

struct smart_ctx {
  smart_config cfg;
  smart_cost cost;
  int device = 0;
  int num_sms = 0;
  int grid_expand = 0, grid_verify = 0, grid_verify_sample = 0;
  size_t select_smem = 0;
  bool fused_select = true;  // selection runs in the layer kernel's last CTA
  bool no_early = false;     // SMART_NO_EARLY=1: every layer kernel waits for the previous grid
  bool in_run_step = false;  // inside smart_run_step: the layer kernels are back to back (early start ok)
  int last_step_grid = 0;    // grid of the step kernel for the last smart_run_step (0: per-layer path)
  // persistent whole-step kernel (step.cu) for smart_run_step: 0 = not usable for this config
  int step_grid = 0;
  size_t step_smem = 0, step_sel_bytes = 0;
  void* step_ws = nullptr;
  double* cost_dev = nullptr;
  Params P{};
  void* ws = nullptr;      // single device allocation
  size_t ws_bytes = 0;
  // host-side call order (graph-capture safe: no device reads)
  int next_layer = 0;      // 0: no step begun
  int phase = 0;           // 0 expect expand, 1 expect select
  bool masked = false;
  cudaStream_t last_stream = nullptr;
  std::string err;
  // NCCL / caller-provided exchange
  void* nccl_comm = nullptr;
  bool byo_exchange = false;
  bool owns_exchange = false;
  // peer exchange (smart_attach_peer_exchange): own send record + device table of receive buffers
  bool peer_exchange = false;
  char* peer_xs = nullptr;
  char** peer_tab = nullptr;
};

namespace {

thread_local std::string g_err;

smart_status fail(smart_ctx* c, smart_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_err = buf;
  return s;
}

#define CUDA_TRY(ctx, call)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return fail(ctx, SMART_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

// ---- NCCL via dlopen ----
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && AllGather && AllReduce && CommDestroy && GetErrorString;
  }
} g_nccl;

long long derive_T(const smart_config* c, int B) {
  long long Wq = c->max_frontier > 0 ? c->max_frontier : (1ll << 30);
  long long t = 1 + std::min<long long>(B, (long long)c->max_depth * Wq);
  if (c->selection == SMART_BASELINE)  // expanded nodes (W per layer) and the final top-B tree
    t = 1 + std::max<long long>(B, (long long)std::max(c->max_depth, 1) * c->max_frontier);
  return c->tree_capacity > 0 ? c->tree_capacity : t;
}

// frontier rows per request per layer: SMART caps them by W and the budget, BASELINE by W only
static long long frontier_width(const smart_config* c, long long B, long long T) {
  long long Wq = c->max_frontier > 0 ? c->max_frontier : (1ll << 30);
  if (c->selection == SMART_BASELINE) return std::max<long long>(1, std::min<long long>(Wq, T - 1));
  return std::max<long long>(1, std::min<long long>(Wq, std::min<long long>(B, T - 1)));
}

smart_status validate(const smart_config* c, const smart_cost* k, smart_sizes* s, std::string& why) {
  auto bad = [&](const char* m) {
    why = m;
    return SMART_EINVAL;
  };
  if (!c) return bad("null config");
  if (c->vocab < 2 || c->vocab > (1 << 24)) return bad("vocab out of range [2, 2^24]");
  if (c->top_k < 1 || c->top_k > 32 || c->top_k > c->vocab) return bad("top_k must be in [1, min(V, 32)]");
  if (c->max_depth < 0 || c->max_depth > SMART_MAX_DEPTH) return bad("max_depth must be in [0, 16]");
  if (c->max_frontier < 0) return bad("max_frontier must be >= 0");
  if (c->batch_local < 1 || c->batch_global < c->batch_local) return bad("batch sizes invalid");
  if (c->batch_offset < 0 || c->batch_offset + c->batch_local > c->batch_global) return bad("batch_offset invalid");
  if (c->batch_global > 65535) return bad("batch_global > 65535");
  if (c->batch_local > 4096) return bad("batch_local > 4096");
  if (!(c->alpha > 0.0 && c->alpha <= 1.0)) return bad("alpha must be in (0, 1]");
  if (c->bonus != 0 && c->bonus != 1) return bad("bonus must be 0 or 1");
  if (c->selection == SMART_BASELINE && (c->max_frontier < 1 || c->batch_local != c->batch_global))
    return bad("BASELINE needs max_frontier >= 1 and a single rank");
  if (c->selection < 0 || c->selection > 2 || c->accept_model < 0 || c->accept_model > 1 || c->marginal < 0 ||
      c->marginal > 1 || c->cost_scope < 0 || c->cost_scope > 1 || c->logits_dtype < 0 || c->logits_dtype > 1 ||
      c->row_mode < 0 || c->row_mode > 2)
    return bad("enum field out of range");
  int B = c->budget_verify / c->batch_global;
  if (B < 1) return bad("per-request budget floor(budget_verify / batch_global) < 1");
  if (k) {
    if (!(k->c_T > 0)) return bad("c_T must be > 0");
    if (k->lambda < 0 || k->gamma < 0 || k->delta < 0 || !(k->rho > 0)) return bad("cost constants out of domain");
    if (!(k->lambda > 0 || (k->gamma > 0 && k->delta > 0))) return bad("marginal cost must be > 0 (lambda > 0 or gamma*delta > 0)");
    if (c->bonus == 1 && k->beta + k->eta <= 0) return bad("bonus = 1 needs beta + eta > 0 (S(empty) finite)");
  }
  long long T = derive_T(c, B);
  if (T < 1 || T > 1024) return bad("tree capacity T must be in [1, 1024]");
  if (c->selection != SMART_BASELINE && c->tree_capacity > 0) {
    // every layer may admit up to min(B - n_r, W) nodes per request, so a tree can hold
    // 1 + min(B, d * W) nodes; a smaller capacity would overflow the per-request arrays
    const long long Wq = c->max_frontier > 0 ? c->max_frontier : (1ll << 30);
    if (T < 1 + std::min<long long>(B, (long long)c->max_depth * Wq))
      return bad("tree_capacity must be >= 1 + min(B, max_depth * max_frontier)");
  }
  long long wf = frontier_width(c, B, T);
  if (c->selection == SMART_BASELINE && T < 1 + std::max<long long>(B, (long long)std::max(c->max_depth, 1) * c->max_frontier))
    return bad("BASELINE tree capacity must hold 1 + max(B, d * W) nodes");
  if (c->selection == SMART_BASELINE &&
      (long long)std::max(c->max_depth, 1) * wf * c->top_k * 16 + T * 4 > 200 * 1024)
    return bad("BASELINE rerank: d * W * k candidates per request exceed shared memory");
  long long cap_rows = (long long)c->batch_local * wf;
  if (cap_rows * c->top_k > 65536ll * 8) return bad("frontier capacity too large");
  if (wf * c->top_k > 65535) return bad("candidates per request exceed 16-bit index");
  int esz = c->logits_dtype == SMART_BF16 ? 2 : 4;
  int ce = kChunkBytes / esz;
  int cpr = (c->vocab + ce - 1) / ce;
  if (cpr > kMaxCpr) return bad("vocab too large for the chunk scheduler (> 64 chunks of 16 KiB per row)");
  if (std::max<long long>(cap_rows, (long long)c->batch_local * T) * cpr >= (1ll << 31))
    return bad("streamed (row, chunk) units exceed 2^31");
  if (s) {
    s->B = B;
    s->T = (int)T;
    s->mask_words = (int)((T + 31) / 32);
    s->frontier_cap = (int)cap_rows;
    s->chunk_elems = ce;
  }
  return SMART_OK;
}

// dynamic shared-memory attributes are per kernel function (process-wide), so every context
// raises them to the largest size any live or earlier context needed; never lowers them
std::mutex g_attr_mu;
size_t g_attr_max[4] = {0, 0, 0, 0};  // mask, walk, rerank, select
cudaError_t raise_attr(int which, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (bytes > g_attr_max[which]) g_attr_max[which] = bytes;
  const size_t v = g_attr_max[which];
  switch (which) {
    case 0: return mask_set_smem_bytes(v);
    case 1: return walk_set_smem_bytes(v);
    case 2: return rerank_set_smem(v);
    default: return select_set_smem(v);
  }
}

// step calls may come from a thread whose current device differs from the context's
inline cudaError_t use_device(const smart_ctx* c) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e == cudaSuccess && cur != c->device) e = cudaSetDevice(c->device);
  return e;
}

int next_pow2(long long n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace

extern "C" {

const char* smart_status_string(smart_status s) {
  switch (s) {
    case SMART_OK: return "ok";
    case SMART_EINVAL: return "invalid argument";
    case SMART_ECUDA: return "CUDA error";
    case SMART_ENCCL: return "NCCL error";
    case SMART_ECAPACITY: return "capacity exceeded";
    case SMART_EDEVICE: return "device flag set (invalid logits)";
    case SMART_ESTATE: return "call out of order";
  }
  return "unknown";
}

const char* smart_last_error(const smart_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

smart_status smart_query_sizes(const smart_config* cfg, smart_sizes* out) {
  std::string why;
  smart_status st = validate(cfg, nullptr, out, why);
  if (st) return fail(nullptr, st, "%s", why.c_str());
  return SMART_OK;
}

// frees everything smart_create may have allocated (used by every failure path after the first
// allocation and by smart_destroy)
static void release_ctx(smart_ctx* c) {
  if (!c) return;
  if (c->ws) cudaFree(c->ws);
  if (c->cost_dev) cudaFree(c->cost_dev);
  if (c->P.dbg) cudaFree(c->P.dbg);
  if (c->step_ws) cudaFree(c->step_ws);
  c->step_ws = nullptr;
  c->ws = nullptr;
  c->cost_dev = nullptr;
  c->P.dbg = nullptr;
  delete c;
}

smart_status smart_create(const smart_config* cfg, const smart_cost* cost, int device, smart_ctx** out) {
  if (!out) return fail(nullptr, SMART_EINVAL, "null out");
  *out = nullptr;
  smart_sizes sz{};
  std::string why;
  smart_status st = validate(cfg, cost, &sz, why);
  if (st) return fail(nullptr, st, "%s", why.c_str());
  if (!cost) return fail(nullptr, SMART_EINVAL, "null cost");

  smart_ctx* c = new smart_ctx();
  c->cfg = *cfg;
  c->cost = *cost;
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete c;
    return fail(nullptr, SMART_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);

  Params& P = c->P;
  P.V = cfg->vocab;
  P.k = cfg->top_k;
  P.d = cfg->max_depth;
  P.Wq = cfg->max_frontier > 0 ? cfg->max_frontier : (1 << 30);
  P.b_loc = cfg->batch_local;
  P.b_glob = cfg->batch_global;
  P.b_off = cfg->batch_offset;
  P.B = sz.B;
  P.T = sz.T;
  P.MW = sz.mask_words;
  P.selection = cfg->selection;
  P.accept_model = cfg->accept_model;
  P.marginal = cfg->marginal;
  P.cost_scope = cfg->cost_scope;
  P.dtype = cfg->logits_dtype;
  P.row_mode = cfg->row_mode;
  P.omega = cfg->bonus;
  P.esz = cfg->logits_dtype == SMART_BF16 ? 2 : 4;
  P.chunk_elems = sz.chunk_elems;
  P.cpr = (P.V + P.chunk_elems - 1) / P.chunk_elems;
  P.cap_rows = sz.frontier_cap;
  P.nranks = 1;
  P.rank = 0;
  P.alpha = cfg->alpha;
  P.lambda = cost->lambda;
  P.beta = cost->beta;
  P.gamma = cost->gamma;
  P.delta = cost->delta;
  P.rho = cost->rho;
  P.eta = cost->eta;
  P.c_T = cost->c_T;

  const long long b = P.b_loc, T = P.T, cap = P.cap_rows, k = P.k, d = std::max(P.d, 1);
  const long long vrows = b * T;
  // exchange sizing (used only with nranks > 1, allocated lazily in attach)
  // workspace carve
  struct Item {
    void** ptr;
    size_t bytes;
  };
  std::vector<Item> items;
  auto add = [&](void* pp, size_t bytes) { items.push_back({reinterpret_cast<void**>(pp), bytes}); };
  add(&P.n_nodes, b * 4);
  add(&P.tok, b * T * 4);
  add(&P.parent, b * T * 4);
  add(&P.depth, b * T * 4);
  add(&P.p, b * T * 4);
  add(&P.cum, b * T * 4);
  add(&P.path_sum, b * T * 8);
  add(&P.E_r, b * 8);
  add(&P.leaf_cnt, b * 4);
  add(&P.leaf_sum, b * 8);
  add(&P.finished, b * 4);
  add(&P.root_pos, b * 4);
  for (int q = 0; q < 2; ++q) {
    add(&P.fr[q], cap * 8);
    add(&P.fr_cum[q], cap * 4);
    add(&P.fr_cnt[q], b * 4);
    add(&P.fr_off[q], b * 4);
    add(&P.fr_total[q], 4);
  }
  add(&P.layer_done, SMART_MAX_DEPTH * 4);
  add(&P.fr_ready, (SMART_MAX_DEPTH + 1) * 4);
  add(&P.cand, d * cap * k * sizeof(Cand));
  add(&P.cand_b, d * cap * k * 4);
  add(&P.cand_adm, d * cap * k * 4);
  add(&P.cand_node, d * cap * k * 4);
  add(&P.cand_rs, d * cap * 8);
  add(&P.trace, SMART_MAX_DEPTH * sizeof(DevTrace));
  add(&P.err, 4);
  add(&P.sum_accept, 16);
  add(&P.sum_glob, 16);
  add(&P.E_glob, 8);
  add(&P.N_glob, 4);
  add(&P.vrow_off, (b + 1) * 4);
  add(&P.vrow_rn, vrows * 8);
  add(&P.vbest, (long long)b * T * 8);
  size_t total = 0;
  for (auto& it : items) total += (it.bytes + 255) & ~size_t(255);
  e = cudaMalloc(&c->ws, total);
  if (e != cudaSuccess) {
    c->ws = nullptr;
    release_ctx(c);
    return fail(nullptr, SMART_ECUDA, "cudaMalloc(%zu): %s", total, cudaGetErrorString(e));
  }
  cudaMemset(c->ws, 0, total);
  c->ws_bytes = total;
  char* base = static_cast<char*>(c->ws);
  for (auto& it : items) {
    *it.ptr = base;
    base += (it.bytes + 255) & ~size_t(255);
  }
  // cost-model tables (fp64, Eqs.(4),(5),(15)): cost(N), marginal(N), N in [0, n_cost)
  {
    const long long wf2 = std::max<long long>(1, std::min<long long>(P.B, T - 1));
    const long long n_cost = (long long)P.b_glob * wf2 + 2;
    std::vector<double> tab(2 * n_cost);
    long long sat_from = (1ll << 62);
    auto costf = [&](double N, bool& sat) {
      double a = cost->delta * std::pow(N, cost->rho);
      if (a > 700.0) { a = 700.0; sat = true; }
      return cost->lambda * N + cost->beta + cost->gamma * (std::exp(a) - 1.0) + cost->eta;
    };
    for (long long N = 0; N < n_cost; ++N) {
      bool sat = false;
      tab[N] = costf((double)N, sat);
      double dcv;
      if (cfg->marginal == SMART_DIFFERENCE) {
        dcv = costf((double)(N + 1), sat) - costf((double)N, sat);
      } else {
        double M = (double)(N < 1 ? 1 : N);
        double a = cost->delta * std::pow(M, cost->rho);
        if (a > 700.0) { a = 700.0; sat = true; }
        dcv = cost->lambda + cost->gamma * cost->delta * cost->rho * std::pow(M, cost->rho - 1.0) * std::exp(a);
      }
      tab[n_cost + N] = dcv;
      if (sat && sat_from > N) sat_from = N;
    }
    e = cudaMalloc(&c->cost_dev, tab.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(c->cost_dev, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      release_ctx(c);
      return fail(nullptr, SMART_ECUDA, "cost table: %s", cudaGetErrorString(e));
    }
    P.cost_tab = c->cost_dev;
    P.dc_tab = c->cost_dev + n_cost;
    P.n_cost = (int)n_cost;
    P.sat_from = sat_from;
  }
  P.min_units = getenv("SMART_MIN_UNITS") ? atoi(getenv("SMART_MIN_UNITS")) : 2;
  if (P.min_units < 1) P.min_units = 1;
  P.debug_mode = getenv("SMART_DEBUG_MODE") ? atoi(getenv("SMART_DEBUG_MODE")) : 0;
  c->no_early = getenv("SMART_NO_EARLY") != nullptr;
  if (getenv("SMART_TIMING")) {
    e = cudaMalloc(&P.dbg, 4096 * sizeof(unsigned long long));
    if (e != cudaSuccess) P.dbg = nullptr;
  }
  // launch geometry: persistent streaming grids sized to the SM count
  c->grid_expand = expand_grid(P.cpr, P.k);
  c->grid_verify = c->num_sms * verify_occupancy();
  c->grid_verify_sample = c->num_sms * verify_occupancy(true);
  // selection: fused into the layer kernel when its scratch fits the stream ring, else the
  // standalone 1024-thread select kernel
  long long elig_cap = b * frontier_width(&c->cfg, P.B, T);
  int sort_cap = next_pow2(std::max<long long>(elig_cap, 1));
  P.sort_cap = sort_cap;
  c->select_smem = select_smem_bytes((int)b, (int)b, sort_cap, (int)(cap * k), 1, (int)k);
  {
    // stage the candidate records in the selection's scratch when it still fits the ring (fused)
    // or the standalone kernel's limit
    const size_t rec = select_rec_bytes((int)(cap * k));
    const size_t lim = c->select_smem <= (size_t)kStages * kChunkBytes ? (size_t)kStages * kChunkBytes : 220 * 1024;
    P.sel_rec = (c->select_smem + rec <= lim) ? 1 : 0;
    if (P.sel_rec) c->select_smem += rec;
  }
  c->fused_select = c->select_smem <= (size_t)kStages * kChunkBytes && c->grid_expand >= 16 && !getenv("SMART_NO_FUSE");
  if (c->select_smem > 220 * 1024) {
    release_ctx(c);
    return fail(nullptr, SMART_ECAPACITY, "selection needs more than 220 KiB of shared memory");
  }
  if (getenv("SMART_VERBOSE"))
    fprintf(stderr, "[smart] grid_expand %d (layer smem %zu B) grid_verify %d select_smem %zu B fused %d\n",
            c->grid_expand, layer_smem_bytes(P.cpr, P.k), c->grid_verify, c->select_smem, (int)c->fused_select);
  // per-step kernels' shared memory is sized from the config at create; a tree capacity whose
  // mask or rerank scratch exceeds the per-CTA limit is a capacity error here, not a launch error
  if (mask_smem_bytes(P.T, P.b_loc) > 227 * 1024 ||
      (P.selection == SMART_BASELINE && rerank_smem_bytes(P) > 227 * 1024)) {
    const int Tcap = P.T;
    release_ctx(c);
    return fail(nullptr, SMART_ECAPACITY, "tree capacity T = %d needs more than 227 KiB of mask/rerank scratch", Tcap);
  }
  e = raise_attr(0, mask_smem_bytes(P.T, P.b_loc));
  if (e == cudaSuccess) e = raise_attr(1, walk_smem_bytes(P.T));
  if (e == cudaSuccess && P.selection == SMART_BASELINE) e = raise_attr(2, rerank_smem_bytes(P));
  if (e == cudaSuccess) e = raise_attr(3, std::max<size_t>(c->select_smem, 48 * 1024));
  if (e != cudaSuccess) {
    release_ctx(c);
    return fail(nullptr, SMART_ECUDA, "shared-memory attributes: %s", cudaGetErrorString(e));
  }
  // persistent whole-step kernel: single rank, SMART selections (PREFIX / FROZEN), node or
  // position pools; its selection CTA always stages the candidate records
  if (P.nranks == 1 && cfg->selection != SMART_BASELINE && cfg->row_mode != SMART_ROWS_FRONTIER &&
      !getenv("SMART_NO_STEP")) {
    c->step_sel_bytes = select_smem_bytes((int)b, (int)b, sort_cap, (int)(cap * k), 1, (int)k) +
                        select_rec_bytes((int)(cap * k));
    c->step_grid = step_grid(P, c->step_sel_bytes, &c->step_smem);
    if (c->step_grid >= 2) {
      const long long S = c->step_grid - 1;
      const long long lists = std::max<long long>(S, std::max<long long>(cap, b));
      const long long rows = std::max<long long>(cap, b);
      const size_t kb = (size_t)lists * k * 16, mb = (size_t)rows * P.cpr * 16, cb = (size_t)rows * k * 16;
      const size_t tb = (size_t)std::max<long long>(cap, b * T) * 8;  // frontier entries, then the verify rows
      auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
      const size_t lines = up(kb) + up(mb) + up(cb);
      e = cudaMalloc(&c->step_ws, lines + up(tb) + sizeof(StepCtl));
      if (e != cudaSuccess) {
        release_ctx(c);
        return fail(nullptr, SMART_ECUDA, "step workspace: %s", cudaGetErrorString(e));
      }
      char* sb = static_cast<char*>(c->step_ws);
      cudaMemset(sb, 0, lines);  // tag 0: never a launch's tag
      P.seg_key = reinterpret_cast<uint4*>(sb);
      sb += up(kb);
      P.seg_ms = reinterpret_cast<uint4*>(sb);
      sb += up(mb);
      P.seg_cand = reinterpret_cast<uint4*>(sb);
      sb += up(cb);
      P.fr_tag = reinterpret_cast<unsigned long long*>(sb);
      cudaMemset(P.fr_tag, 0, tb);
      sb += up(tb);
      P.ctl = reinterpret_cast<StepCtl*>(sb);
      cudaMemset(P.ctl, 0, sizeof(StepCtl));
    } else {
      c->step_grid = 0;
    }
  }
  if (getenv("SMART_VERBOSE"))
    fprintf(stderr, "[smart] step kernel grid %d smem %zu B (selection scratch %zu B)\n", c->step_grid, c->step_smem,
            c->step_sel_bytes);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    release_ctx(c);
    return fail(nullptr, SMART_ECUDA, "init: %s", cudaGetErrorString(e));
  }
  *out = c;
  return SMART_OK;
}

smart_status smart_nccl_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(nullptr, SMART_EINVAL, "null id");
  if (!g_nccl.load()) return fail(nullptr, SMART_ENCCL, "cannot dlopen libnccl.so.2");
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, SMART_ENCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(id_out, &id, 128);
  return SMART_OK;
}

static long long exchange_record_bytes(long long b_loc, long long wf) {
  const long long m_cap = b_loc * wf;
  return (m_cap * 8 + b_loc * 8 + (b_loc + 2) * 4 + 255) & ~255ll;
}

static smart_status setup_exchange(smart_ctx* c, int rank, int nranks, void* send, void* recv) {
  Params& P = c->P;
  P.nranks = nranks;
  P.rank = rank;
  const long long b = P.b_loc;
  const long long wf = frontier_width(&c->cfg, P.B, P.T);
  P.m_cap = (int)(b * wf);
  P.xstride = exchange_record_bytes(b, wf);
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->owns_exchange) {
    cudaFree(P.xs);
    cudaFree(P.xr);
  }
  if (send && recv) {
    P.xs = static_cast<char*>(send);
    P.xr = static_cast<char*>(recv);
    c->owns_exchange = false;
  } else {
    CUDA_TRY(c, cudaMalloc(&P.xs, P.xstride));
    CUDA_TRY(c, cudaMalloc(&P.xr, P.xstride * nranks));
    c->owns_exchange = true;
  }
  CUDA_TRY(c, cudaMemset(P.xs, 0, P.xstride));
  const int sort_cap = next_pow2((long long)P.m_cap * nranks);
  P.sort_cap = sort_cap;
  size_t need = select_smem_bytes((int)b, (int)P.b_glob, sort_cap, P.cap_rows * P.k, nranks, P.k);
  const size_t rec = select_rec_bytes(P.cap_rows * P.k);
  P.sel_rec = (need + rec <= 220 * 1024) ? 1 : 0;
  if (P.sel_rec) need += rec;
  if (need > 220 * 1024) return fail(c, SMART_ECAPACITY, "global selection needs %zu B shared memory", need);
  c->select_smem = std::max(c->select_smem, need);
  c->fused_select = false;
  CUDA_TRY(c, raise_attr(3, std::max<size_t>(c->select_smem, 48 * 1024)));
  return SMART_OK;
}

static smart_status check_sharding(smart_ctx* c, int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, SMART_EINVAL, "bad rank/nranks");
  if (c->cfg.batch_local * nranks != c->cfg.batch_global || c->cfg.batch_offset != rank * c->cfg.batch_local)
    return fail(c, SMART_EINVAL, "sharding must be equal contiguous ranges: offset = rank * batch_local");
  if (nranks > 1 && c->cfg.cost_scope != SMART_COST_GLOBAL)
    return fail(c, SMART_EINVAL, "LOCAL cost scope needs no exchange");
  return SMART_OK;
}

smart_status smart_attach_nccl(smart_ctx* c, const uint8_t id[128], int rank, int nranks) {
  if (!c || !id) return fail(c, SMART_EINVAL, "null argument");
  smart_status st = check_sharding(c, rank, nranks);
  if (st) return st;
  if (nranks == 1) return SMART_OK;
  if (!g_nccl.load()) return fail(c, SMART_ENCCL, "cannot dlopen libnccl.so.2");
  CUDA_TRY(c, cudaSetDevice(c->device));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = g_nccl.CommInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) return fail(c, SMART_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
  c->nccl_comm = comm;
  return setup_exchange(c, rank, nranks, nullptr, nullptr);
}

smart_status smart_exchange_record_bytes(const smart_config* cfg, int nranks, int64_t* bytes) {
  smart_sizes sz{};
  std::string why;
  smart_status st = validate(cfg, nullptr, &sz, why);
  if (st) return fail(nullptr, st, "%s", why.c_str());
  if (!bytes || nranks < 1) return fail(nullptr, SMART_EINVAL, "bad argument");
  const long long Wq = cfg->max_frontier > 0 ? cfg->max_frontier : (1ll << 30);
  const long long wf = std::max<long long>(1, std::min<long long>(Wq, std::min<long long>(sz.B, sz.T - 1)));
  *bytes = exchange_record_bytes(cfg->batch_local, wf);
  return SMART_OK;
}

smart_status smart_attach_exchange(smart_ctx* c, int rank, int nranks, void* d_send, void* d_recv) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  if (!d_send || !d_recv) return fail(c, SMART_EINVAL, "null exchange buffers");
  if ((reinterpret_cast<uintptr_t>(d_send) | reinterpret_cast<uintptr_t>(d_recv)) & 255)
    return fail(c, SMART_EINVAL, "exchange buffers must be 256-byte aligned");
  smart_status st = check_sharding(c, rank, nranks);
  if (st) return st;
  c->byo_exchange = true;
  return setup_exchange(c, rank, nranks, d_send, d_recv);
}

smart_status smart_peer_exchange_bytes(const smart_config* cfg, int nranks, int64_t* bytes) {
  int64_t rec = 0;
  smart_status st = smart_exchange_record_bytes(cfg, nranks, &rec);
  if (st) return st;
  *bytes = rec * nranks + ((8ll * nranks + 255) & ~255ll);  // records, then one tag word per rank
  return SMART_OK;
}

smart_status smart_attach_peer_exchange(smart_ctx* c, int rank, int nranks, void* const* d_recv_bufs) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  if (!d_recv_bufs) return fail(c, SMART_EINVAL, "null receive-buffer table");
  for (int g = 0; g < nranks; ++g)
    if (!d_recv_bufs[g] || (reinterpret_cast<uintptr_t>(d_recv_bufs[g]) & 255))
      return fail(c, SMART_EINVAL, "receive buffer %d null or not 256-byte aligned", g);
  smart_status st = check_sharding(c, rank, nranks);
  if (st) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (!c->peer_xs) {
    int64_t rec = 0;
    st = smart_exchange_record_bytes(&c->cfg, nranks, &rec);
    if (st) return st;
    CUDA_TRY(c, cudaMalloc(&c->peer_xs, (size_t)rec));
  }
  st = setup_exchange(c, rank, nranks, c->peer_xs, d_recv_bufs[rank]);
  if (st) return st;
  if (c->peer_tab) cudaFree(c->peer_tab);
  CUDA_TRY(c, cudaMalloc(&c->peer_tab, sizeof(char*) * nranks));
  CUDA_TRY(c, cudaMemcpy(c->peer_tab, d_recv_bufs, sizeof(char*) * nranks, cudaMemcpyHostToDevice));
  c->P.xpeer = c->peer_tab;
  c->P.xtag_off = c->P.xstride * nranks;
  c->byo_exchange = true;
  c->peer_exchange = true;
  return SMART_OK;
}

smart_status smart_ipc_get_handle(void* d_ptr, uint8_t handle[64]) {
  if (!d_ptr || !handle) return fail(nullptr, SMART_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, d_ptr);
  if (e != cudaSuccess) return fail(nullptr, SMART_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  memcpy(handle, &h, 64);
  return SMART_OK;
}

smart_status smart_ipc_open_handle(const uint8_t handle[64], void** d_ptr) {
  if (!d_ptr || !handle) return fail(nullptr, SMART_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  const cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(nullptr, SMART_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  return SMART_OK;
}

smart_status smart_ipc_close(void* d_ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  if (e != cudaSuccess) return fail(nullptr, SMART_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return SMART_OK;
}

smart_status smart_destroy(smart_ctx* c) {
  if (!c) return SMART_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->peer_xs) cudaFree(c->peer_xs);
  if (c->peer_tab) cudaFree(c->peer_tab);
  if (c->nccl_comm && g_nccl.h) g_nccl.CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  if (c->owns_exchange) {
    cudaFree(c->P.xs);
    cudaFree(c->P.xr);
  }
  release_ctx(c);
  return SMART_OK;
}

smart_status smart_begin_step(smart_ctx* c, const int32_t* d_root_tok, const int32_t* d_root_pos, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int thr = 256, grid = (c->P.b_loc + thr - 1) / thr;
  launch_k(begin_step_kernel, dim3(grid), dim3(thr), 0, s, c->P, d_root_tok, d_root_pos);
  CUDA_TRY(c, cudaGetLastError());
  ++c->P.xepoch;  // the peer-exchange tags of this step
  c->next_layer = 1;
  c->phase = 0;
  c->masked = false;
  c->last_stream = s;
  return SMART_OK;
}

smart_status smart_expand_step(smart_ctx* c, int32_t layer, const void* d_logits, int64_t ld, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  if (!d_logits) return fail(c, SMART_EINVAL, "null logits");
  if (ld < c->cfg.vocab) return fail(c, SMART_EINVAL, "ld (%lld) < vocab (%d)", (long long)ld, c->cfg.vocab);
  if (c->next_layer == 0) return fail(c, SMART_ESTATE, "expand before begin_step");
  if (layer != c->next_layer || c->phase != 0 || layer > c->cfg.max_depth)
    return fail(c, SMART_ESTATE, "expand layer %d out of order (expected %d, phase %d)", layer, c->next_layer, c->phase);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long ld_bytes = (long long)ld * c->P.esz;
  // TMA bulk copies need 16-byte aligned rows and 16-byte multiple row lengths
  const bool tma = ((reinterpret_cast<uintptr_t>(d_logits) & 15) == 0) && (ld_bytes % 16 == 0) &&
                   (((long long)c->P.V * c->P.esz) % 16 == 0);
  // early start: the previous layer's fused selection publishes its frontier before its kernel ends
  // (only inside smart_run_step: between separate calls the caller may run its own kernels, e.g.
  // a draft forward writing these logits, which the flag does not order against)
  const bool early = layer >= 2 && c->in_run_step && c->fused_select && c->P.nranks <= 1 && !c->no_early;
  launch_expand(c->P, layer, d_logits, ld_bytes, tma, c->fused_select, early, c->grid_expand, s);
  CUDA_TRY(c, cudaGetLastError());
  c->phase = 1;
  c->last_stream = s;
  return SMART_OK;
}

smart_status smart_select(smart_ctx* c, int32_t layer, int32_t* d_frontier, int32_t* d_frontier_count, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  if (layer != c->next_layer || c->phase != 1)
    return fail(c, SMART_ESTATE, "select layer %d out of order (expected %d after expand)", layer, c->next_layer);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->byo_exchange && c->P.nranks > 1) {
    launch_select(c->P, layer, 1 /* kSelLocal */, c->select_smem, s);
    if (c->peer_exchange) launch_peer_push(c->P, layer, s);  // the record into every rank's buffer
    CUDA_TRY(c, cudaGetLastError());
    c->phase = 2;  // awaiting smart_select_finish (after the caller's all-gather, or the peer pushes)
    c->last_stream = s;
    return SMART_OK;
  }
  if (c->P.nranks > 1) {
    launch_select(c->P, layer, 1 /* kSelLocal */, c->select_smem, s);
    CUDA_TRY(c, cudaGetLastError());
    ncclResult_t r = g_nccl.AllGather(c->P.xs, c->P.xr, (size_t)c->P.xstride, ncclUint8,
                                      static_cast<ncclComm_t>(c->nccl_comm), s);
    if (r != ncclSuccess) return fail(c, SMART_ENCCL, "ncclAllGather: %s", g_nccl.GetErrorString(r));
    launch_select(c->P, layer, 2 /* kSelGlobal */, c->select_smem, s);
  } else if (!c->fused_select) {
    launch_select(c->P, layer, 0 /* kSelFull */, c->select_smem, s);
  }  // else: already done by the layer kernel's last CTA
  CUDA_TRY(c, cudaGetLastError());
  if (d_frontier || d_frontier_count) launch_export_frontier(c->P, layer & 1, d_frontier, d_frontier_count, s);
  CUDA_TRY(c, cudaGetLastError());
  c->next_layer = layer + 1;
  c->phase = 0;
  c->last_stream = s;
  return SMART_OK;
}

smart_status smart_select_finish(smart_ctx* c, int32_t layer, int32_t* d_frontier, int32_t* d_frontier_count,
                                 void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  if (layer != c->next_layer || c->phase != 2)
    return fail(c, SMART_ESTATE, "select_finish layer %d out of order", layer);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->peer_exchange) launch_peer_wait(c->P, layer, s);  // every rank's record has landed
  launch_select(c->P, layer, 2 /* kSelGlobal */, c->select_smem, s);
  CUDA_TRY(c, cudaGetLastError());
  if (d_frontier || d_frontier_count) launch_export_frontier(c->P, layer & 1, d_frontier, d_frontier_count, s);
  CUDA_TRY(c, cudaGetLastError());
  c->next_layer = layer + 1;
  c->phase = 0;
  c->last_stream = s;
  return SMART_OK;
}

smart_status smart_build_mask(smart_ctx* c, uint32_t* d_mask, int32_t* d_pos, int32_t* d_parent, int32_t* d_tok,
                              int32_t* d_tree_len, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  if (c->next_layer == 0 || c->phase != 0) return fail(c, SMART_ESTATE, "build_mask needs a begun step between layers");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->P.selection == SMART_BASELINE) launch_rerank(c->P, s);  // stage 2 of the baseline (Q32)
  launch_mask(c->P, d_mask, d_pos, d_parent, d_tok, d_tree_len, s);
  CUDA_TRY(c, cudaGetLastError());
  c->masked = true;
  c->last_stream = s;
  return SMART_OK;
}

// C2: the end-of-step sums (accept lengths, drafted nodes) over all ranks for the
// global acceptance rate beta = sum a / sum n, one NCCL all-reduce of two u64 on the
// step's stream when a communicator is attached; otherwise the local sums are copied
static smart_status end_of_step(smart_ctx* c, cudaStream_t s) {
  if (c->nccl_comm && c->P.nranks > 1) {
    ncclResult_t r = g_nccl.AllReduce(c->P.sum_accept, c->P.sum_glob, 2, ncclUint64, ncclSum,
                                      static_cast<ncclComm_t>(c->nccl_comm), s);
    if (r != ncclSuccess) return fail(c, SMART_ENCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
  } else {
    CUDA_TRY(c, cudaMemcpyAsync(c->P.sum_glob, c->P.sum_accept, 16, cudaMemcpyDeviceToDevice, s));
  }
  return SMART_OK;
}

smart_status smart_verify_accept(smart_ctx* c, const void* d_target, int64_t ld, int32_t* d_accept_len,
                                 int32_t* d_accept_path, int32_t* d_bonus, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  if (!d_target) return fail(c, SMART_EINVAL, "null target logits");
  if (ld < c->cfg.vocab) return fail(c, SMART_EINVAL, "ld < vocab");
  if (!c->masked) return fail(c, SMART_ESTATE, "verify_accept must follow build_mask");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long ld_bytes = (long long)ld * c->P.esz;
  const bool tma = ((reinterpret_cast<uintptr_t>(d_target) & 15) == 0) && (ld_bytes % 16 == 0) &&
                   (((long long)c->P.V * c->P.esz) % 16 == 0);
  launch_verify(c->P, d_target, ld_bytes, tma, d_accept_len, d_accept_path, d_bonus, c->grid_verify, s);
  CUDA_TRY(c, cudaGetLastError());
  c->last_stream = s;
  return end_of_step(c, s);
}

smart_status smart_verify_sample(smart_ctx* c, const void* d_target, int64_t ld, double temperature, uint64_t seed,
                                 int32_t* d_accept_len, int32_t* d_accept_path, int32_t* d_bonus, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, use_device(c));
  if (!d_target) return fail(c, SMART_EINVAL, "null target logits");
  if (ld < c->cfg.vocab) return fail(c, SMART_EINVAL, "ld < vocab");
  if (!(temperature > 0.0) || !(1.0 / temperature < 3.0e38)) return fail(c, SMART_EINVAL, "temperature must be > 0");
  if (!c->masked) return fail(c, SMART_ESTATE, "verify_sample must follow build_mask");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long ld_bytes = (long long)ld * c->P.esz;
  const bool tma = ((reinterpret_cast<uintptr_t>(d_target) & 15) == 0) && (ld_bytes % 16 == 0) &&
                   (((long long)c->P.V * c->P.esz) % 16 == 0);
  launch_verify(c->P, d_target, ld_bytes, tma, d_accept_len, d_accept_path, d_bonus, c->grid_verify_sample, s, true,
                (float)(1.0 / temperature), (unsigned long long)seed);
  CUDA_TRY(c, cudaGetLastError());
  c->last_stream = s;
  return end_of_step(c, s);
}

smart_status smart_run_step(smart_ctx* c, const int32_t* d_root_tok, const int32_t* d_root_pos, const void* d_draft,
                            int64_t ld, const void* d_target, int64_t ld_t, uint32_t* d_mask, int32_t* d_pos,
                            int32_t* d_parent, int32_t* d_tok, int32_t* d_tree_len, int32_t* d_accept_len,
                            int32_t* d_accept_path, int32_t* d_bonus, void* stream) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  if (c->cfg.row_mode == SMART_ROWS_FRONTIER)
    return fail(c, SMART_EINVAL, "smart_run_step needs row_mode NODE or POSITION (pre-filled pools)");
  if (c->byo_exchange && !c->peer_exchange)
    return fail(c, SMART_ESTATE, "smart_run_step cannot drive a caller-provided exchange");
  if (!d_draft) return fail(c, SMART_EINVAL, "null draft logits");
  if (ld < c->cfg.vocab || (d_target && ld_t < c->cfg.vocab)) return fail(c, SMART_EINVAL, "ld < vocab");
  if (c->step_grid > 0 && c->P.nranks <= 1) {
    // one persistent launch for the whole step (step.cu) when both pools are TMA-addressable
    const long long ldb = (long long)ld * c->P.esz, ldtb = (long long)ld_t * c->P.esz;
    const bool rb = (((long long)c->P.V * c->P.esz) % 16) == 0;
    const bool tma = rb && ((reinterpret_cast<uintptr_t>(d_draft) & 15) == 0) && (ldb % 16 == 0) &&
                     (!d_target || (((reinterpret_cast<uintptr_t>(d_target) & 15) == 0) && (ldtb % 16 == 0)));
    if (tma) {
      CUDA_TRY(c, use_device(c));
      cudaStream_t s = static_cast<cudaStream_t>(stream);
      StepOut o{d_mask, d_pos, d_parent, d_tok, d_tree_len, d_accept_len, d_accept_path, d_bonus};
      launch_step(c->P, c->step_grid, c->step_smem, c->step_sel_bytes, d_draft, ldb, d_target, ldtb, d_root_tok,
                  d_root_pos, o, s);
      CUDA_TRY(c, cudaGetLastError());
      c->last_step_grid = c->step_grid;
      c->next_layer = c->cfg.max_depth + 1;
      c->phase = 0;
      c->masked = true;
      c->last_stream = s;
      return d_target ? end_of_step(c, s) : SMART_OK;
    }
  }
  c->last_step_grid = 0;
  smart_status st = smart_begin_step(c, d_root_tok, d_root_pos, stream);
  c->in_run_step = true;
  for (int l = 1; !st && l <= c->cfg.max_depth; ++l) {
    st = smart_expand_step(c, l, d_draft, ld, stream);
    if (!st) st = smart_select(c, l, nullptr, nullptr, stream);
    if (!st && c->phase == 2) st = smart_select_finish(c, l, nullptr, nullptr, stream);  // peer exchange
  }
  c->in_run_step = false;
  if (!st) st = smart_build_mask(c, d_mask, d_pos, d_parent, d_tok, d_tree_len, stream);
  if (!st && d_target) st = smart_verify_accept(c, d_target, ld_t, d_accept_len, d_accept_path, d_bonus, stream);
  return st;
}

extern "C" int smart_debug_probes(smart_ctx* c, unsigned long long* host16, int reset) {
  if (!c || !c->P.dbg) return -1;
  cudaStreamSynchronize(c->last_stream);
  if (host16) cudaMemcpy(host16, c->P.dbg, 4096 * 8, cudaMemcpyDeviceToHost);
  if (reset) {
    static unsigned long long init[4096];
    for (int i = 0; i < 4096; ++i)  // reset 2: all zero (step-kernel probes use max / ~min slots)
      init[i] = (reset != 2 && (i == 0 || i == 8 || (i >= 64 && !(i & 1)))) ? ~0ull : 0ull;
    cudaMemcpy(c->P.dbg, init, sizeof init, cudaMemcpyHostToDevice);
  }
  return 0;
}

smart_status smart_get_stats(smart_ctx* c, smart_stats* out) {
  if (!c || !out) return fail(c, SMART_EINVAL, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  DevTrace tr[SMART_MAX_DEPTH];
  int err = 0;
  unsigned long long acc = 0, glob[2] = {0, 0};
  double E = 0;
  int N = 0;
  CUDA_TRY(c, cudaMemcpy(tr, c->P.trace, sizeof tr, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(&err, c->P.err, 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(&acc, c->P.sum_accept, 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(glob, c->P.sum_glob, 16, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(&E, c->P.E_glob, 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(&N, c->P.N_glob, 4, cudaMemcpyDeviceToHost));
  std::vector<int> nn(c->P.b_loc);
  CUDA_TRY(c, cudaMemcpy(nn.data(), c->P.n_nodes, 4 * nn.size(), cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof *out);
  out->error_flags = err;
  out->accepted_local = (int64_t)acc;
  long long nodes = 0;
  for (int v : nn) nodes += v - 1;
  out->nodes_local = nodes;
  out->step_kernel_grid = c->last_step_grid;
  out->accepted_global = (int64_t)glob[0];
  out->nodes_global = (int64_t)glob[1];
  out->E_global = E;
  int le = 0;
  for (int l = 0; l < SMART_MAX_DEPTH; ++l) {
    smart_layer_trace& t = out->layer[l];
    t.executed = tr[l].executed;
    t.n_rows = tr[l].n_rows;
    t.n_cand = tr[l].n_cand;
    t.n_elig = tr[l].n_elig;
    t.n_admit = tr[l].n_admit;
    t.argmax_j = tr[l].argmax_j;
    t.N0 = tr[l].N0;
    t.saturated = tr[l].saturated;
    t.select_path = tr[l].select_path;
    t.n_screened = tr[l].n_screened;
    t.E0 = tr[l].E0;
    t.S0 = tr[l].S0;
    t.S_after = tr[l].S_after;
    t.dc0 = tr[l].dc0;
    if (t.executed) {
      le = l + 1;
      out->S_final = t.S_after;
    }
  }
  out->layers_executed = le;
  if (le == 0) {
    // no layer ran: S of the root-only batch
    int bc = c->cfg.cost_scope == SMART_COST_LOCAL ? c->P.b_loc : c->P.b_glob;
    double C = c->cost.lambda * 0 + c->cost.beta + c->cost.eta;
    out->S_final = C > 0 ? c->cost.c_T * (c->P.omega * bc) / (bc * C) : 0.0;
  }
  if (err & (kErrDraftNaN | kErrTargetNaN)) return fail(c, SMART_EDEVICE, "invalid logits (NaN/+inf) seen (flags %d)", err);
  if (err & kErrTimeout) return fail(c, SMART_EDEVICE, "a device-side wait timed out (flags %d)", err);
  return SMART_OK;
}

smart_status smart_get_tree(smart_ctx* c, int32_t* n_nodes, int32_t* tok, int32_t* parent, int32_t* depth, float* p,
                            float* cum) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  size_t bt = (size_t)c->P.b_loc * c->P.T;
  if (n_nodes) CUDA_TRY(c, cudaMemcpy(n_nodes, c->P.n_nodes, 4 * c->P.b_loc, cudaMemcpyDeviceToHost));
  if (tok) CUDA_TRY(c, cudaMemcpy(tok, c->P.tok, 4 * bt, cudaMemcpyDeviceToHost));
  if (parent) CUDA_TRY(c, cudaMemcpy(parent, c->P.parent, 4 * bt, cudaMemcpyDeviceToHost));
  if (depth) CUDA_TRY(c, cudaMemcpy(depth, c->P.depth, 4 * bt, cudaMemcpyDeviceToHost));
  if (p) CUDA_TRY(c, cudaMemcpy(p, c->P.p, 4 * bt, cudaMemcpyDeviceToHost));
  if (cum) CUDA_TRY(c, cudaMemcpy(cum, c->P.cum, 4 * bt, cudaMemcpyDeviceToHost));
  return SMART_OK;
}

smart_status smart_get_candidates(smart_ctx* c, int32_t layer, int64_t cap, int32_t* count, int32_t* ints,
                                  float* floats, int32_t* admitted) {
  if (!c) return fail(nullptr, SMART_EINVAL, "null ctx");
  if (layer < 1 || layer > std::max(c->cfg.max_depth, 1)) return fail(c, SMART_EINVAL, "layer out of range");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->last_stream));
  DevTrace tr;
  CUDA_TRY(c, cudaMemcpy(&tr, c->P.trace + (layer - 1), sizeof tr, cudaMemcpyDeviceToHost));
  int rows = tr.executed ? tr.n_rows : 0;
  const int k = c->P.k;
  long long n = (long long)rows * k;
  if (count) *count = (int32_t)n;
  if (n > cap) return fail(c, SMART_EINVAL, "cap %lld < %lld candidates", (long long)cap, n);
  if (n == 0) return SMART_OK;
  size_t lb = (size_t)(layer - 1) * c->P.cap_rows * k;
  std::vector<Cand> cd(n);
  std::vector<float> bb(n);
  std::vector<int> adm(n);
  CUDA_TRY(c, cudaMemcpy(cd.data(), c->P.cand + lb, n * sizeof(Cand), cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(bb.data(), c->P.cand_b + lb, n * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(adm.data(), c->P.cand_adm + lb, n * 4, cudaMemcpyDeviceToHost));
  std::vector<int2> rs(rows);
  CUDA_TRY(c, cudaMemcpy(rs.data(), c->P.cand_rs + (size_t)(layer - 1) * c->P.cap_rows, rows * sizeof(int2),
                         cudaMemcpyDeviceToHost));
  for (long long q = 0; q < n; ++q) {
    const int2 e = rs[q / k];
    if (ints) {
      ints[q * 4 + 0] = e.x;
      ints[q * 4 + 1] = cd[q].parent;
      ints[q * 4 + 2] = cd[q].tok;
      ints[q * 4 + 3] = e.y * k + (int)(q % k);
    }
    if (floats) {
      floats[q * 3 + 0] = cd[q].p;
      floats[q * 3 + 1] = cd[q].cum;
      floats[q * 3 + 2] = bb[q];
    }
    if (admitted) admitted[q] = adm[q];
  }
  return SMART_OK;
}

}  // extern "C"
