// select.cu — standalone K2 `smart_select` kernel: one CTA of 1024 threads running
// select_layer (select_core.cuh).  Used when the selection cannot be fused into the layer
// kernel's last CTA: sharded batches (phase kSelLocal -> NCCL all-gather -> phase kSelGlobal)
// and batches whose selection scratch exceeds the layer kernel's shared-memory ring.
#include "select_core.cuh"

namespace smart {

namespace {

__global__ void __launch_bounds__(kSelectThreads, 1) select_kernel(Params P, int layer, int mode) {
  extern __shared__ __align__(16) char smem[];
  const int par = (layer - 1) & 1;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) P.layer_done[layer - 1] = 0;  // row arrivals of the layer kernel (unused here)
  if (mode == kSelFull && *P.fr_total[par] == 0) {
    // no frontier: the step has terminated; publish an empty next frontier
    if (threadIdx.x == 0) *P.fr_total[layer & 1] = 0;
    return;
  }
  tl_start(P, 40 + layer);
  select_layer<kSelectThreads>(P, layer, mode, smem, NoWait{}, PubReady{&P.fr_ready[layer]});
  tl_end(P, 40 + layer);
  if (SMART_PROBES && P.dbg) {  // this layer's clock64 phase stamps (select_layer's stamp() slots)
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 9; j <= 22; ++j) P.dbg[3000 + layer * 16 + (j - 9)] = P.dbg[32 + j];
  }
}

__global__ void export_frontier_kernel(Params P, int parity, int32_t* out, int32_t* count) {
  pdl_wait();
  pdl_trigger();
  const int n = *P.fr_total[parity];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; out && i < n; i += gridDim.x * blockDim.x) {
    const int2 e = P.fr[parity][i];
    out[2 * i] = e.x;
    out[2 * i + 1] = e.y;
  }
  if (count && blockIdx.x == 0 && threadIdx.x == 0) *count = n;
}

}  // namespace

size_t select_smem_bytes(int b_loc, int b_all, int sort_cap, int nc_cap, int nranks, int k) {
  return sel_smem_bytes(b_loc, b_all, sort_cap, nc_cap, nranks, k);
}

size_t select_rec_bytes(int nc_cap) { return sel_rec_bytes(nc_cap); }

cudaError_t select_set_smem(size_t bytes) {
  cudaFuncSetAttribute(select_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(export_frontier_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  return cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ---- peer exchange (NEXT #4): the local phase's record written straight into every
// rank's receive buffer, then one tag word per (rank -> receiver) with release semantics at system
// scope; the receiver polls the tags of all ranks (acquire) before its global phase.  Tags carry
// (step counter << 32 | layer), so a stale record is never accepted and nothing is reset. ----
__device__ __forceinline__ unsigned long long peer_tag(const Params& P, int layer) {
  return (P.xepoch << 32) | (unsigned)layer;
}
__global__ void __launch_bounds__(256) peer_push_kernel(Params P, int layer) {
  const int tid = threadIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(P.xs);
  const int n16 = (int)(P.xstride / 16);
  for (int g = 0; g < P.nranks; ++g) {
    uint4* dst = reinterpret_cast<uint4*>(P.xpeer[g] + (size_t)P.rank * P.xstride);
    for (int i = tid; i < n16; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (tid < P.nranks) {  // release (cumulative over the barrier): the record before the tag
    unsigned long long* tg = reinterpret_cast<unsigned long long*>(P.xpeer[tid] + P.xtag_off) + P.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(tg), "l"(peer_tag(P, layer)) : "memory");
  }
}
__global__ void __launch_bounds__(32) peer_wait_kernel(Params P, int layer) {
  const int g = threadIdx.x;
  if (g < P.nranks) {
    const unsigned long long* tg = reinterpret_cast<const unsigned long long*>(P.xr + P.xtag_off) + g;
    const unsigned long long want = peer_tag(P, layer);
    for (unsigned it = 0;; ++it) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(tg) : "memory");
      if (v == want) break;
      if (it > (1u << 24)) {  // a rank that never pushes: sticky flag instead of a hang
        atomicOr(P.err, kErrTimeout);
        break;
      }
      __nanosleep(64);
    }
  }
}
void launch_peer_push(const Params& P, int layer, cudaStream_t s) { peer_push_kernel<<<1, 256, 0, s>>>(P, layer); }
void launch_peer_wait(const Params& P, int layer, cudaStream_t s) { peer_wait_kernel<<<1, 32, 0, s>>>(P, layer); }

void launch_select(const Params& P, int layer, int mode, size_t smem, cudaStream_t s) {
  launch_k(select_kernel, dim3(1), dim3(kSelectThreads), smem, s, P, layer, mode);
}

void launch_export_frontier(const Params& P, int parity, int32_t* d_frontier, int32_t* d_count, cudaStream_t s) {
  if (d_frontier) launch_k(export_frontier_kernel, dim3(8), dim3(256), 0, s, P, parity, d_frontier, d_count);
  else if (d_count) launch_k(export_frontier_kernel, dim3(1), dim3(32), 0, s, P, parity, (int32_t*)nullptr, d_count);
}

}  // namespace smart
