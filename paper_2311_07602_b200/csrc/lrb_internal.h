// lrb_internal.h — context object and helpers shared by the C-ABI units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/lrb.h"

struct lrb_ctx {
  int device = 0;
  int sm_count = 148;
  size_t l2_bytes = 0;
  int variant_override = -1;
  int loader_override = -1;  // -1 auto, 0 segment copies, 1 TMA tensor maps (when eligible)
  std::string err;
  std::atomic<uint64_t> launches{0};
  uint64_t capture_launches0 = 0;  // launch counter at lrb_graph_begin
  // host-buffer pipeline: per-lane stream and device staging buffers
  static constexpr int kLanes = 3;
  cudaStream_t lane_stream[kLanes] = {nullptr, nullptr, nullptr};
  double* lane_buf[kLanes] = {nullptr, nullptr, nullptr};
  size_t lane_bytes[kLanes] = {0, 0, 0};
  // pointer-array plans: one auxiliary stream per variant group so the groups'
  // persistent grids overlap their tails (fork/join through events)
  static constexpr int kAux = 4;
  cudaStream_t aux_stream[kAux] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t aux_done[kAux] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr;
  // stream-ordered scratch pool (keeps freed blocks for reuse instead of
  // returning them to the driver at every synchronisation)
  cudaMemPool_t pool = nullptr;
  // L2 flush buffer
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
};

namespace lrb {

void set_error(lrb_ctx* ctx, const char* fmt, ...);
lrb_status fail(lrb_ctx* ctx, lrb_status st, const char* fmt, ...);
lrb_status cuda_fail(lrb_ctx* ctx, cudaError_t e, const char* where);
lrb_status bind(lrb_ctx* ctx);  // cudaSetDevice(ctx->device)

}  // namespace lrb

#define LRB_CUDA_TRY(ctx, call)                                   \
  do {                                                            \
    cudaError_t lrb_e_ = (call);                                  \
    if (lrb_e_ != cudaSuccess) return lrb::cuda_fail(ctx, lrb_e_, #call); \
  } while (0)
