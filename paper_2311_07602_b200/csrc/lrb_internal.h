// lrb_internal.h — context object and helpers shared by the C-ABI units.
#pragma once

#include <cuda.h>
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
  int last_variant = -1;  // kernel of the last strided GEMM (lrb_last_variant)
  int loader_override = -1;  // -1 auto, 0 segment copies, 1 TMA tensor maps (when eligible)
  std::string err;
  std::atomic<uint64_t> launches{0};
  uint64_t capture_launches0 = 0;  // launch counter at lrb_graph_begin
  // host-buffer pipeline: per-lane stream and device staging buffers
  static constexpr int kLanes = 3;
  cudaStream_t lane_stream[kLanes] = {nullptr, nullptr, nullptr};
  double* lane_buf[kLanes] = {nullptr, nullptr, nullptr};
  size_t lane_bytes[kLanes] = {0, 0, 0};
  // pageable host buffers: per-lane pinned staging (inputs / outputs) and the
  // events that say when a lane's staging can be reused
  void* lane_hin[kLanes] = {nullptr, nullptr, nullptr};
  size_t lane_hin_bytes[kLanes] = {0, 0, 0};
  void* lane_hout[kLanes] = {nullptr, nullptr, nullptr};
  size_t lane_hout_bytes[kLanes] = {0, 0, 0};
  cudaEvent_t lane_h2d[kLanes] = {nullptr, nullptr, nullptr};
  cudaEvent_t lane_d2h[kLanes] = {nullptr, nullptr, nullptr};
  // pointer-array plans: one auxiliary stream per variant group so the groups'
  // persistent grids overlap their tails (fork/join through events)
  static constexpr int kAux = 4;
  cudaStream_t aux_stream[kAux] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t aux_done[kAux] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr;
  // stream-ordered scratch pool (keeps freed blocks for reuse instead of
  // returning them to the driver at every synchronisation)
  cudaMemPool_t pool = nullptr;
  // grow-only workspace for multi-launch paths (low-rank r > 32): allocated
  // outside stream capture, so a captured graph references it instead of
  // carrying alloc/free memory nodes; ws_ev orders consecutive eager users
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t ws_ev = nullptr;
  bool ws_pending = false;
  // outgrown workspaces: a captured graph may still reference them, so they
  // are released only by lrb_destroy (after the device is idle)
  std::vector<void*> ws_retired;
  // L2 flush buffer
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
};

namespace lrb {

void set_error(lrb_ctx* ctx, const char* fmt, ...);
lrb_status fail(lrb_ctx* ctx, lrb_status st, const char* fmt, ...);
lrb_status cuda_fail(lrb_ctx* ctx, cudaError_t e, const char* where);
lrb_status bind(lrb_ctx* ctx);  // cudaSetDevice(ctx->device)
// context workspace of >= bytes, ordered after its previous eager user on
// another stream. It grows only outside stream capture; a capture that needs
// more gets a stream-ordered (graph-owned) allocation instead (*temporary).
lrb_status acquire_workspace(lrb_ctx* ctx, size_t bytes, cudaStream_t s, void** out,
                             bool* temporary);
void release_workspace(lrb_ctx* ctx, cudaStream_t s, void* p, bool temporary);
// the auxiliary streams / fork-join events, created on first use
lrb_status ensure_aux(lrb_ctx* ctx);
// Host side of the host-buffer pipelines. Pinned buffers are copied with
// cudaMemcpyAsync directly; pageable ones through the lane's pinned staging
// with a multi-threaded memcpy (the driver's own pageable path runs ~10 GB/s).
// Per call: begin(l) before reusing lane l, h2d/d2h for each operand, then
// inputs_done(l) / outputs_done(l), and finish() at the end.
class HostPipe {
 public:
  HostPipe(lrb_ctx* ctx, int lanes) : ctx_(ctx), lanes_(lanes) {}
  // staging sizes per lane (bytes); only allocated when a buffer is pageable
  lrb_status prepare(size_t in_bytes, size_t out_bytes);
  lrb_status begin(int lane);
  lrb_status h2d(int lane, void* dev, const void* host, size_t bytes);
  lrb_status inputs_done(int lane);
  lrb_status d2h(int lane, void* host, const void* dev, size_t bytes);
  lrb_status outputs_done(int lane);
  lrb_status finish();

 private:
  struct Pending {
    void* dst;
    size_t off, bytes;
  };
  lrb_ctx* ctx_;
  int lanes_;
  size_t in_off_[lrb_ctx::kLanes] = {0, 0, 0}, out_off_[lrb_ctx::kLanes] = {0, 0, 0};
  bool used_in_[lrb_ctx::kLanes] = {false, false, false};
  std::vector<Pending> pend_[lrb_ctx::kLanes];
};
bool host_pinned(const void* p);
int debug_flags();  // LRB_DEBUG_FLAGS probe bits (lrb_api.cu)
// tensor maps (lrb_api.cu): a (rows, cols, z) column-major operand with box
// (box_in, box_out, 1); the 4-D reconstruction output map (x, y, j, i) of an
// n x n row-major matrix of b x b tiles, box 16 x nb, 128-byte swizzle.
// False when TMA's alignment rules are not met.
bool encode_operand(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                    int64_t stride, int64_t zdim, int box_in, int box_out);
bool encode_tiles_c_map(CUtensorMap* map, double* out, int64_t n, int64_t b, int nb);
void par_memcpy(void* dst, const void* src, size_t bytes);
// stream-ordered allocation from the context pool (blocks stay mapped)
inline cudaError_t pool_alloc(lrb_ctx* ctx, void** p, size_t bytes, cudaStream_t s) {
  return ctx->pool ? cudaMallocFromPoolAsync(p, bytes, ctx->pool, s) : cudaMallocAsync(p, bytes, s);
}

}  // namespace lrb

#define LRB_CUDA_TRY(ctx, call)                                   \
  do {                                                            \
    cudaError_t lrb_e_ = (call);                                  \
    if (lrb_e_ != cudaSuccess) return lrb::cuda_fail(ctx, lrb_e_, #call); \
  } while (0)
