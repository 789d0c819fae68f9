// lrb_host.cu — host side of the host-buffer pipelines: pinned-buffer
// detection, multi-threaded staging copies and the per-lane pipeline state.
//
// The host-buffer entry points (lrb_dgemm_strided_batched_host,
// lrb_lowrank_multiply_host) move a batch through the device in chunks on the
// context's lane streams. From pinned memory the copies are plain
// cudaMemcpyAsync calls and run at PCIe speed. Pageable memory would make the
// driver stage through its own buffers one copy at a time (~10 GB/s here);
// instead each lane owns pinned staging, filled and drained by several host
// threads while the copy engines work on the other lanes.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "lrb_internal.h"

namespace lrb {

bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = size_t(4) << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t parts = std::min<size_t>(std::min<size_t>(hw, 16), (bytes + kPiece - 1) / kPiece);
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes + parts - 1) / parts;
  std::vector<std::thread> pool;
  pool.reserve(parts - 1);
  for (size_t i = 1; i < parts; ++i) {
    const size_t b = std::min(bytes, i * per), e = std::min(bytes, b + per);
    pool.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
    });
  }
  std::memcpy(dst, src, std::min(bytes, per));
  for (auto& t : pool) t.join();
}

lrb_status HostPipe::prepare(size_t in_bytes, size_t out_bytes) {
  for (int l = 0; l < lanes_; ++l) {
    if (!ctx_->lane_h2d[l]) {
      LRB_CUDA_TRY(ctx_, cudaEventCreateWithFlags(&ctx_->lane_h2d[l], cudaEventDisableTiming));
      LRB_CUDA_TRY(ctx_, cudaEventCreateWithFlags(&ctx_->lane_d2h[l], cudaEventDisableTiming));
    }
    if (in_bytes > ctx_->lane_hin_bytes[l]) {
      if (ctx_->lane_hin[l]) cudaFreeHost(ctx_->lane_hin[l]);
      ctx_->lane_hin[l] = nullptr;
      ctx_->lane_hin_bytes[l] = 0;
      LRB_CUDA_TRY(ctx_, cudaMallocHost(&ctx_->lane_hin[l], in_bytes));
      ctx_->lane_hin_bytes[l] = in_bytes;
    }
    if (out_bytes > ctx_->lane_hout_bytes[l]) {
      if (ctx_->lane_hout[l]) cudaFreeHost(ctx_->lane_hout[l]);
      ctx_->lane_hout[l] = nullptr;
      ctx_->lane_hout_bytes[l] = 0;
      LRB_CUDA_TRY(ctx_, cudaMallocHost(&ctx_->lane_hout[l], out_bytes));
      ctx_->lane_hout_bytes[l] = out_bytes;
    }
  }
  return LRB_OK;
}

lrb_status HostPipe::begin(int l) {
  // the lane's previous chunk: its staged inputs must have reached the device
  // and its staged outputs must be drained before the staging is reused
  if (used_in_[l]) LRB_CUDA_TRY(ctx_, cudaEventSynchronize(ctx_->lane_h2d[l]));
  if (!pend_[l].empty()) {
    LRB_CUDA_TRY(ctx_, cudaEventSynchronize(ctx_->lane_d2h[l]));
    for (const Pending& p : pend_[l])
      par_memcpy(p.dst, static_cast<char*>(ctx_->lane_hout[l]) + p.off, p.bytes);
    pend_[l].clear();
  }
  used_in_[l] = false;
  in_off_[l] = out_off_[l] = 0;
  return LRB_OK;
}

lrb_status HostPipe::h2d(int l, void* dev, const void* host, size_t bytes) {
  if (!bytes) return LRB_OK;
  cudaStream_t s = ctx_->lane_stream[l];
  if (host_pinned(host)) {
    LRB_CUDA_TRY(ctx_, cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
    return LRB_OK;
  }
  if (in_off_[l] + bytes > ctx_->lane_hin_bytes[l])
    return fail(ctx_, LRB_ERR_CAPACITY, "host pipeline: input staging too small");
  char* stage = static_cast<char*>(ctx_->lane_hin[l]) + in_off_[l];
  par_memcpy(stage, host, bytes);
  LRB_CUDA_TRY(ctx_, cudaMemcpyAsync(dev, stage, bytes, cudaMemcpyHostToDevice, s));
  in_off_[l] += (bytes + 255) / 256 * 256;
  used_in_[l] = true;
  return LRB_OK;
}

lrb_status HostPipe::inputs_done(int l) {
  if (used_in_[l]) LRB_CUDA_TRY(ctx_, cudaEventRecord(ctx_->lane_h2d[l], ctx_->lane_stream[l]));
  return LRB_OK;
}

lrb_status HostPipe::d2h(int l, void* host, const void* dev, size_t bytes) {
  if (!bytes) return LRB_OK;
  cudaStream_t s = ctx_->lane_stream[l];
  if (host_pinned(host)) {
    LRB_CUDA_TRY(ctx_, cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
    return LRB_OK;
  }
  if (out_off_[l] + bytes > ctx_->lane_hout_bytes[l])
    return fail(ctx_, LRB_ERR_CAPACITY, "host pipeline: output staging too small");
  char* stage = static_cast<char*>(ctx_->lane_hout[l]) + out_off_[l];
  LRB_CUDA_TRY(ctx_, cudaMemcpyAsync(stage, dev, bytes, cudaMemcpyDeviceToHost, s));
  pend_[l].push_back({host, out_off_[l], bytes});
  out_off_[l] += (bytes + 255) / 256 * 256;
  return LRB_OK;
}

lrb_status HostPipe::outputs_done(int l) {
  if (!pend_[l].empty())
    LRB_CUDA_TRY(ctx_, cudaEventRecord(ctx_->lane_d2h[l], ctx_->lane_stream[l]));
  return LRB_OK;
}

lrb_status HostPipe::finish() {
  for (int l = 0; l < lanes_; ++l) {
    LRB_CUDA_TRY(ctx_, cudaStreamSynchronize(ctx_->lane_stream[l]));
    for (const Pending& p : pend_[l])
      par_memcpy(p.dst, static_cast<char*>(ctx_->lane_hout[l]) + p.off, p.bytes);
    pend_[l].clear();
  }
  return LRB_OK;
}

}  // namespace lrb
