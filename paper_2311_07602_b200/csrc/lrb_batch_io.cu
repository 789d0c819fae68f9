// lrb_batch_io.cu — LRBATCH1 batch files straight to / from device memory.
//
// Format (reference proj/include/lrbatch/batch_io.hpp:11-24): magic
// "LRBATCH1", then little-endian uint64 batch_size, block_size, rank_a,
// rank_b, then the four LowRankBatch role arrays back to back (a_vt, b_u,
// a_x, b_x) as little-endian doubles; results are not stored. Errors and
// their texts follow save_batch / load_batch (batch_io.hpp:29-77): IoError
// for open/write failures, ParseError for bad magic and truncation.
//
// The device loader streams the payload through two pinned staging buffers:
// the file read of chunk c+1 overlaps the H2D copy of chunk c.
#include <cstdio>
#include <cstring>
#include <string>

#include "lrb_internal.h"

using lrb::fail;

namespace {

constexpr char kMagic[8] = {'L', 'R', 'B', 'A', 'T', 'C', 'H', '1'};
constexpr size_t kStage = size_t(32) << 20;  // 32 MiB pinned staging buffers

struct File {
  FILE* f = nullptr;
  explicit File(FILE* p) : f(p) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

lrb_status read_header(lrb_ctx* ctx, FILE* f, const std::string& path, int64_t hdr[4]) {
  char magic[8];
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
    return fail(ctx, LRB_ERR_PARSE, "not a batch file (bad magic): %s", path.c_str());
  uint64_t v[4];
  if (std::fread(v, 8, 4, f) != 4)
    return fail(ctx, LRB_ERR_PARSE, "truncated batch header: %s", path.c_str());
  for (int i = 0; i < 4; ++i) hdr[i] = int64_t(v[i]);
  // LowRankBatch constructor invariants (low_rank.hpp:123-133)
  if (v[0] < 1 || v[1] < 1 || v[2] < 1 || v[3] < 1)
    return fail(ctx, LRB_ERR_SHAPE, "LowRankBatch: degenerate dimensions in %s", path.c_str());
  return LRB_OK;
}

// element counts of the four roles
void role_counts(const int64_t hdr[4], int64_t n[4]) {
  n[0] = hdr[0] * hdr[2] * hdr[1];  // a_vt: rank_a x block
  n[1] = hdr[0] * hdr[1] * hdr[3];  // b_u: block x rank_b
  n[2] = hdr[0] * hdr[2] * hdr[2];  // a_x
  n[3] = hdr[0] * hdr[3] * hdr[3];  // b_x
}

}  // namespace

extern "C" lrb_status lrb_batch_file_header(const char* path, int64_t* hdr) {
  if (!path || !hdr) return fail(nullptr, LRB_ERR_ARG, "lrb_batch_file_header: null argument");
  File in(std::fopen(path, "rb"));
  if (!in.f) return fail(nullptr, LRB_ERR_IO, "cannot open for reading: %s", path);
  return read_header(nullptr, in.f, path, hdr);
}

extern "C" lrb_status lrb_batch_file_load(lrb_ctx* ctx, const char* path, double* a_vt,
                                          double* b_u, double* a_x, double* b_x, int device_ptrs) {
  if (!path) return fail(ctx, LRB_ERR_ARG, "lrb_batch_file_load: null path");
  File in(std::fopen(path, "rb"));
  if (!in.f) return fail(ctx, LRB_ERR_IO, "cannot open for reading: %s", path);
  int64_t hdr[4];
  lrb_status st = read_header(ctx, in.f, path, hdr);
  if (st) return st;
  int64_t n[4];
  role_counts(hdr, n);
  double* dst[4] = {a_vt, b_u, a_x, b_x};
  for (int r = 0; r < 4; ++r)
    if (!dst[r]) return fail(ctx, LRB_ERR_ARG, "lrb_batch_file_load: role %d buffer is null", r);
  if (!device_ptrs) {
    for (int r = 0; r < 4; ++r)
      if (std::fread(dst[r], 8, size_t(n[r]), in.f) != size_t(n[r]))
        return fail(ctx, LRB_ERR_PARSE, "truncated batch payload: %s", path);
    return LRB_OK;
  }
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "lrb_batch_file_load: null ctx");
  st = lrb::bind(ctx);
  if (st) return st;
  // double-buffered pinned staging: read chunk c+1 while chunk c copies
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaStream_t s = ctx->lane_stream[0];
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    for (int i = 0; i < 2; ++i) {
      if (stage[i]) cudaFreeHost(stage[i]);
      if (done[i]) cudaEventDestroy(done[i]);
    }
  };
  for (int i = 0; i < 2; ++i) {
    cudaError_t e = cudaMallocHost(&stage[i], kStage);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      cleanup();
      return lrb::cuda_fail(ctx, e, "lrb_batch_file_load: staging");
    }
  }
  int buf = 0;
  bool used[2] = {false, false};
  for (int r = 0; r < 4; ++r) {
    size_t left = size_t(n[r]) * 8, off = 0;
    char* d = reinterpret_cast<char*>(dst[r]);
    while (left) {
      const size_t chunk = std::min(left, kStage);
      if (used[buf]) cudaEventSynchronize(done[buf]);  // staging buffer free again
      if (std::fread(stage[buf], 1, chunk, in.f) != chunk) {
        cleanup();
        return fail(ctx, LRB_ERR_PARSE, "truncated batch payload: %s", path);
      }
      cudaError_t e = cudaMemcpyAsync(d + off, stage[buf], chunk, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaEventRecord(done[buf], s);
      if (e != cudaSuccess) {
        cleanup();
        return lrb::cuda_fail(ctx, e, "lrb_batch_file_load: copy");
      }
      used[buf] = true;
      buf ^= 1;
      off += chunk;
      left -= chunk;
    }
  }
  cleanup();
  return LRB_OK;
}

extern "C" lrb_status lrb_batch_file_save(lrb_ctx* ctx, const char* path, int64_t batch,
                                          int64_t block, int64_t rank_a, int64_t rank_b,
                                          const double* a_vt, const double* b_u,
                                          const double* a_x, const double* b_x, int device_ptrs) {
  if (!path) return fail(ctx, LRB_ERR_ARG, "lrb_batch_file_save: null path");
  if (batch < 1 || block < 1 || rank_a < 1 || rank_b < 1)
    return fail(ctx, LRB_ERR_SHAPE, "LowRankBatch: degenerate dimensions");
  const double* src[4] = {a_vt, b_u, a_x, b_x};
  for (int r = 0; r < 4; ++r)
    if (!src[r]) return fail(ctx, LRB_ERR_ARG, "lrb_batch_file_save: role %d buffer is null", r);
  if (device_ptrs) {
    if (!ctx) return fail(nullptr, LRB_ERR_ARG, "lrb_batch_file_save: null ctx");
    lrb_status st = lrb::bind(ctx);
    if (st) return st;
  }
  File out(std::fopen(path, "wb"));
  if (!out.f) return fail(ctx, LRB_ERR_IO, "cannot open for writing: %s", path);
  const int64_t hdr[4] = {batch, block, rank_a, rank_b};
  bool ok = std::fwrite(kMagic, 1, 8, out.f) == 8;
  for (int i = 0; i < 4 && ok; ++i) {
    const uint64_t v = uint64_t(hdr[i]);
    ok = std::fwrite(&v, 8, 1, out.f) == 1;
  }
  int64_t n[4];
  role_counts(hdr, n);
  void* stage = nullptr;
  if (ok && device_ptrs && cudaMallocHost(&stage, kStage) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, LRB_ERR_CAPACITY, "lrb_batch_file_save: pinned staging");
  }
  // the role buffers may still be written by work on non-blocking streams
  // (e.g. lrb_fill_uniform on a context stream), which the legacy-stream
  // copies below would not wait for: let all device work finish first
  if (ok && device_ptrs && cudaDeviceSynchronize() != cudaSuccess) {
    cudaFreeHost(stage);
    return lrb::cuda_fail(ctx, cudaGetLastError(), "lrb_batch_file_save: device sync");
  }
  for (int r = 0; r < 4 && ok; ++r) {
    if (!device_ptrs) {
      ok = std::fwrite(src[r], 8, size_t(n[r]), out.f) == size_t(n[r]);
      continue;
    }
    size_t left = size_t(n[r]) * 8, off = 0;
    const char* sp = reinterpret_cast<const char*>(src[r]);
    while (left && ok) {
      const size_t chunk = std::min(left, kStage);
      ok = cudaMemcpy(stage, sp + off, chunk, cudaMemcpyDeviceToHost) == cudaSuccess &&
           std::fwrite(stage, 1, chunk, out.f) == chunk;
      off += chunk;
      left -= chunk;
    }
  }
  if (stage) cudaFreeHost(stage);
  if (!ok) return fail(ctx, LRB_ERR_IO, "write failed: %s", path);
  return LRB_OK;
}
