// lrb_varn.h — the single-launch variable-size pointer-array kernel
// (lrb_varn.cu): problem descriptor and launch entry shared with the planner.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lrb {

struct ItemDesc;  // lrb_gemm.cuh

constexpr int kVarnMB = 128;    // rows of C per tile (4 warps x 32)
constexpr int kVarnNB = 64;     // max columns of C per tile
// (overridable at build time for A/B probes: -DLRB_VARN_KB=16 -DLRB_VARN_STAGES=4)
#ifndef LRB_VARN_KB
#define LRB_VARN_KB 32
#endif
#ifndef LRB_VARN_STAGES
#define LRB_VARN_STAGES 2
#endif
constexpr int kVarnKB = LRB_VARN_KB;          // k chunk per ring slot
constexpr int kVarnStages = LRB_VARN_STAGES;  // ring depth (two CTAs per SM)
// TMA box width (columns) of an op(B) = N operand for an item with n
// columns: the tile's columns rounded up to the DMMA fragment width
__host__ __device__ __forceinline__ int varn_box_cols(int n) {
  const int c = n < kVarnNB ? n : kVarnNB;
  return (c + 7) / 8 * 8;
}

struct VarnProblem {
  const ItemDesc* items;
  const uint64_t* tiles;       // (item << 32) | (ti << 16) | tj, in claim order; or null:
  const CUtensorMap* maps;     // 2 per item (A, B), 3-D with z extent 1
  int64_t num_tiles;           // (host-built tile list)
  unsigned long long* next;    // [0] ticket counter, [1] finished CTAs (self-resetting)
  // device-built plans (tiles == null): tickets index the tiles of the
  // ordered items through their exclusive tile prefix
  const int64_t* prefix;       // [count + 1]
  const uint32_t* order;       // [count] item ids, claim order
  const unsigned int* count;   // number of ordered items
  const int64_t* total;        // prefix[count]
  const uint64_t* dev_tiles;   // the expanded tile list, valid when *total <= dev_cap
  long long dev_cap;
};

// Position p of ticket t in an exclusive prefix (prefix[p] <= t <
// prefix[p + 1], p < count). Tickets a CTA takes only grow, so the search
// runs forward from its previous position (*cursor): exponential, then binary.
__device__ __forceinline__ int64_t prefix_search(const int64_t* prefix, int64_t count, int64_t t,
                                                 int64_t* cursor) {
  int64_t p = *cursor;
  if (p >= count || prefix[p] > t) p = 0;
  int64_t step = 1, hi = p + 1;
  while (hi < count && prefix[hi] <= t) {
    p = hi;
    step *= 2;
    hi = p + step;
  }
  if (hi > count) hi = count;
  while (hi - p > 1) {
    const int64_t mid = (p + hi) / 2;
    if (prefix[mid] <= t)
      p = mid;
    else
      hi = mid;
  }
  *cursor = p;
  return p;
}

// order generic-proxy writes of a tensor map in global memory (another
// kernel's tensormap.replace, or a copy) before TMA reads through it
__device__ __forceinline__ void fence_tensormap_acquire(const void* map) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(map) : "memory");
}

// a_t / b_t: op flags of the column-major view; flags bit 0: beta = 1
cudaError_t launch_varn(int a_t, int b_t, const VarnProblem& p, int flags, int device,
                        int sm_count, cudaStream_t stream, int64_t* grid);

}  // namespace lrb
