// Selection-CTA microbenchmark: select_layer (select_core.cuh) of one cfg3-shaped layer (32
// requests x 1 row x k = 8 candidates, layer 1) on one CTA of the step kernel's shape (8 warps),
// alone on the GPU; prints the clock64 phase stamps (build with -DSMART_PROBES=1).
//   mode 0: default path; mode 1: SMART_DEBUG_MODE 7 (threshold path off)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSMART_PROBES=1 -I include
//          -I paper_2604_09731_b200/csrc tools/ubench/select.cu -o /tmp/selbench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "select_core.cuh"

using namespace smart;

struct NoPub {
  __device__ void operator()(int) const {}
  __device__ void entry(int, int, int) const {}
};

__global__ void __launch_bounds__(288, 1) sel_bench(Params P, const int4* recs, int R) {
  extern __shared__ __align__(128) char dsm[];
  const int tid = threadIdx.x;
  if (tid >= 256) return;
  const int k = P.k;
  auto wait_rows = [&](SelLayout& L, int4* crec) -> bool {
    for (int q = tid; q < R * k; q += 256) crec[q] = recs[q];
    for (int row = tid; row < R; row += 256) L.rreq[row] = row;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    return true;
  };
  const long long t0 = clock64();
  select_layer<256>(P, 1, kSelFull, dsm, wait_rows, NoPub{});
  asm volatile("bar.sync 1, 256;" ::: "memory");
  if (tid == 0) P.dbg[0] = clock64() - t0;
}

template <class T>
T* dalloc(size_t n, T v = T()) {
  std::vector<T> h(n, v);
  T* d = nullptr;
  cudaMalloc(&d, n * sizeof(T));
  cudaMemcpy(d, h.data(), n * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}

int main(int argc, char** argv) {
  const int b = 32, k = 8, W = 8, d = 6, Bv = 200, T = 8;
  const int R = b, cap_rows = b * 8;
  Params P{};
  P.V = 128256; P.k = k; P.d = d; P.Wq = W; P.b_loc = b; P.b_glob = b; P.b_off = 0; P.B = Bv / b; P.T = T;
  P.MW = 1; P.selection = SMART_PREFIX; P.accept_model = SMART_NODE_SUM; P.marginal = SMART_DERIVATIVE;
  P.cost_scope = SMART_COST_GLOBAL; P.omega = 1; P.cap_rows = cap_rows; P.nranks = 1;
  // cfg3 cost (roofline fixture of the sharding test): lam, gamma, delta, rho, eta = c_T
  const double lam = 0.0084, gam = 6.69, del = 6.3e-7, rho = 2.23, eta = 2.47;
  P.alpha = 0.8; P.lambda = lam; P.gamma = gam; P.delta = del; P.rho = rho; P.eta = eta; P.c_T = eta;
  const int ncost = 4096;
  std::vector<double> ct(ncost), dt(ncost);
  for (int N = 0; N < ncost; ++N) {
    const double a = del * pow((double)N, rho);
    ct[N] = lam * N + gam * (exp(a) - 1.0) + eta;
    const double Nm = N < 1 ? 1.0 : (double)N;
    dt[N] = lam + gam * del * rho * pow(Nm, rho - 1.0) * exp(del * pow(Nm, rho));
  }
  double* dct = dalloc<double>(ncost);
  double* ddt = dalloc<double>(ncost);
  cudaMemcpy(dct, ct.data(), ncost * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ddt, dt.data(), ncost * 8, cudaMemcpyHostToDevice);
  P.cost_tab = dct; P.dc_tab = ddt; P.n_cost = ncost; P.sort_cap = 256; P.sel_rec = 1; P.sat_from = 1ll << 40;
  P.n_nodes = dalloc<int>(b, 1); P.tok = dalloc<int>(b * T); P.parent = dalloc<int>(b * T); P.depth = dalloc<int>(b * T);
  P.p = dalloc<float>(b * T); P.cum = dalloc<float>(b * T); P.path_sum = dalloc<double>(b * T);
  P.E_r = dalloc<double>(b); P.leaf_cnt = dalloc<int>(b, 1); P.leaf_sum = dalloc<double>(b);
  P.finished = dalloc<int>(b); P.root_pos = dalloc<int>(b);
  std::vector<int> off(b);
  for (int r = 0; r < b; ++r) off[r] = r;
  for (int q = 0; q < 2; ++q) {
    P.fr[q] = dalloc<int2>(cap_rows); P.fr_cum[q] = dalloc<float>(cap_rows);
    P.fr_cnt[q] = dalloc<int>(b, 1); P.fr_off[q] = dalloc<int>(b); P.fr_total[q] = dalloc<int>(1, b);
    cudaMemcpy(P.fr_off[q], off.data(), b * 4, cudaMemcpyHostToDevice);
  }
  P.cand = dalloc<Cand>(d * cap_rows * k); P.cand_b = dalloc<float>(d * cap_rows * k);
  P.cand_adm = dalloc<int>(d * cap_rows * k); P.cand_node = dalloc<int>(d * cap_rows * k);
  P.cand_rs = dalloc<int2>(d * cap_rows);
  P.trace = dalloc<DevTrace>(SMART_MAX_DEPTH); P.err = dalloc<int>(1);
  P.sum_accept = dalloc<unsigned long long>(2); P.E_glob = dalloc<double>(1); P.N_glob = dalloc<int>(1);
  P.dbg = dalloc<unsigned long long>(4096);
  // candidates: per row p sorted desc (top-1 ~0.6, a tail like the synthetic draft rows)
  std::vector<int4> rec(R * k);
  srand(7);
  for (int row = 0; row < R; ++row) {
    double rem = 1.0;
    for (int h = 0; h < k; ++h) {
      const double f = h == 0 ? 0.45 + 0.3 * (rand() / (double)RAND_MAX) : 0.02 + 0.05 * (rand() / (double)RAND_MAX);
      const float p = (float)(rem * f);
      rem -= rem * f;
      int pi;
      memcpy(&pi, &p, 4);
      rec[row * k + h] = make_int4(1000 + h, pi, pi, 0);
    }
  }
  int4* drec = dalloc<int4>(R * k);
  cudaMemcpy(drec, rec.data(), R * k * 16, cudaMemcpyHostToDevice);
  const size_t smem = sel_smem_bytes(b, b, 256, cap_rows * k, 1, k) + (size_t)cap_rows * k * 16;
  cudaFuncSetAttribute(sel_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[23] = {0};
  names[9] = "start"; names[10] = "benefits"; names[11] = "req-rank"; names[12] = "sort"; names[13] = "A5 cut";
  names[15] = "bitmaps"; names[16] = "B6"; names[20] = "popc"; names[21] = "scan"; names[17] = "counts";
  names[18] = "frontier"; names[19] = "published"; names[14] = "adm flags"; names[22] = "end";
  const int order[] = {9, 10, 11, 12, 13, 15, 16, 20, 21, 17, 18, 19, 14, 22};
  for (int mode = 0; mode < 2; ++mode) {
    P.debug_mode = mode == 1 ? 7 : 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(P.dbg, 0, 4096 * 8);
      cudaMemcpy(P.n_nodes, std::vector<int>(b, 1).data(), b * 4, cudaMemcpyHostToDevice);
      cudaMemset(P.finished, 0, b * 4);
      cudaMemset(P.E_r, 0, b * 8);
      cudaMemset(P.N_glob, 0, 4);
      sel_bench<<<1, 288, smem>>>(P, drec, R);
      cudaDeviceSynchronize();
    }
    unsigned long long h[64];
    cudaMemcpy(h, P.dbg, sizeof h, cudaMemcpyDeviceToHost);
    DevTrace tr;
    cudaMemcpy(&tr, P.trace, sizeof tr, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): total %llu cycles; elig %d admit %d argmax %d |", mode, mode ? "block path" : "default",
           h[0], tr.n_elig, tr.n_admit, tr.argmax_j);
    for (int s : order)
      if (h[32 + s]) printf(" %s %lld", names[s], (long long)(h[32 + s] - h[32 + 9]));
    printf("\n");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
