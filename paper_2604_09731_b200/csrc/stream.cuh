// stream.cuh — TMA-staged persistent streaming of logit rows (B200, sm_100a).
//
// A persistent grid of CTAs, each = 1 producer warp + kConsumerWarps consumer warps.  Every CTA
// owns a balanced contiguous range of (row, 16 KiB chunk) units.  The producer's elected lane
// issues 1-D bulk copies (cp.async.bulk global -> shared, completion on an mbarrier with a
// transaction count) into a kStages-deep ring; consumers wait on the stage's "full" barrier,
// pull their 16-byte vectors out of shared memory and release the stage on its "empty"
// barrier.  With 6 stages x 16 KiB per CTA and 2 CTAs per SM, up to 192 KiB per SM is in
// flight — a small layer (32 rows = 8 MiB) is entirely in flight after one DRAM latency.
#pragma once

#include "smart_internal.cuh"

namespace smart {

constexpr int kStages = 5;
constexpr int kMinUnits = 4;   // chunks per CTA at least (64 KiB, all in flight)
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;      // 256 consumer threads
constexpr int kLayerThreads = kConsumers + 32;       // + 1 producer warp
static_assert(kConsumers == kStreamThreads, "consumer slice mapping assumes 256 consumers");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)  // suspend-time hint (ns): sleep in hardware instead of re-polling
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine; SASS UBLKCP), completes tx bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// named barrier among the consumer warps only (the producer warp may have exited)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

template <int S>
struct StreamPipeT {
  uint64_t full[S];
  uint64_t empty[S];
};
using StreamPipe = StreamPipeT<kStages>;

// smem layout of a streaming CTA: [ring kStages x 16 KiB][pipe][kernel-specific]
struct RowRange {
  int lo, hi;  // [lo, hi) of the (row, chunk) units, row-major; totals < 2^31 (checked at create)
};

// balanced contiguous ranges over min(gridDim.x, ceil(total / min_units)) CTAs (32-bit integer
// math only): small layers use fewer CTAs with several chunks each, all in flight in the ring
__device__ __forceinline__ RowRange cta_range_min(int total, int min_units) {
  int g = (total + min_units - 1) / min_units;
  if (g > (int)gridDim.x) g = (int)gridDim.x;
  RowRange r;
  const int b = (int)blockIdx.x;
  if (b >= g) {
    r.lo = r.hi = 0;
    return r;
  }
  const int base = total / g, rem = total - base * g;
  r.lo = b * base + min(b, rem);
  r.hi = r.lo + base + (b < rem ? 1 : 0);
  return r;
}

// Producer loop (one elected lane): stream chunks [lo, hi) of rows whose base pointer is given
// by `row_base(row)`; each row is `row_bytes` long (16-byte multiple).  (row, chunk) advance
// incrementally (no division per chunk).
template <int S, class RowBase>
__device__ __forceinline__ void produce(StreamPipeT<S>& pipe, char* ring, RowRange rr, int cpr, long long row_bytes,
                                        RowBase row_base) {
  int row = rr.lo / cpr, c = rr.lo - row * cpr;
  const char* base = row_base(row);
  int i = 0;
  for (int q = rr.lo; q < rr.hi; ++q, ++i) {
    const int s = i % S;
    const uint32_t n = (uint32_t)(i / S);
    mbar_wait(&pipe.empty[s], (n & 1u) ^ 1u);
    const long long off = (long long)c * kChunkBytes;
    const uint32_t bytes = (uint32_t)min((long long)kChunkBytes, row_bytes - off);
    mbar_expect_tx(&pipe.full[s], bytes);
    bulk_g2s(ring + (size_t)s * kChunkBytes, base + off, bytes, &pipe.full[s]);
    if (++c == cpr) {
      c = 0;
      if (q + 1 < rr.hi) base = row_base(++row);
    }
  }
}

}  // namespace smart
