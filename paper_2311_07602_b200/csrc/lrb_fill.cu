// lrb_fill.cu — on-device synthetic operand generation with the counter RNG of
// include/lrb_rng.h (bit-identical to the host oracle's generator), so shards
// and chunks regenerate their slice of a batch from global item indices.
#include <vector>

#include "../../include/lrb_rng.h"
#include "lrb_internal.h"

namespace {

// blockIdx.y strides over items, x over the column-major elements of an item.
__global__ void fill_strided_kernel(double* __restrict__ dst, int64_t rows, int64_t cols, int64_t ld,
                                    int64_t stride, int64_t batch, uint64_t key, int64_t item0) {
  const int64_t per = rows * cols;
  for (int64_t item = blockIdx.y; item < batch; item += gridDim.y) {
    double* d = dst + item * stride;
    const uint64_t gi = uint64_t(item0 + item);
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < per;
         e += int64_t(gridDim.x) * blockDim.x) {
      const int64_t c = e / rows, r = e - c * rows;
      d[c * ld + r] = lrb_uniform(key, gi, uint64_t(e));
    }
  }
}

struct FillDesc {
  double* dst;
  int64_t rows, cols, ld;
};

__global__ void fill_ptr_kernel(const FillDesc* __restrict__ desc, int64_t batch, uint64_t key,
                                int64_t item0) {
  for (int64_t item = blockIdx.y; item < batch; item += gridDim.y) {
    const FillDesc f = desc[item];
    const int64_t per = f.rows * f.cols;
    const uint64_t gi = uint64_t(item0 + item);
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < per;
         e += int64_t(gridDim.x) * blockDim.x) {
      const int64_t c = e / f.rows, r = e - c * f.rows;
      f.dst[c * f.ld + r] = lrb_uniform(key, gi, uint64_t(e));
    }
  }
}

}  // namespace

using lrb::fail;

extern "C" lrb_status lrb_fill_uniform(lrb_ctx* ctx, double* dst, int64_t rows, int64_t cols,
                                       int64_t ld, int64_t stride, int64_t batch, uint64_t seed,
                                       uint32_t role, int64_t item_offset, void* stream) {
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "lrb_fill_uniform: null ctx");
  if (rows < 0 || cols < 0 || batch < 0 || item_offset < 0)
    return fail(ctx, LRB_ERR_SHAPE, "lrb_fill_uniform: negative size");
  if (rows * cols > (int64_t(1) << 32))
    return fail(ctx, LRB_ERR_UNSUPPORTED, "lrb_fill_uniform: more than 2^32 elements per item");
  if (ld < std::max<int64_t>(1, rows))
    return fail(ctx, LRB_ERR_SHAPE, "lrb_fill_uniform: ld is %lld but rows is %lld", (long long)ld,
                (long long)rows);
  if (batch > 1 && rows * cols > 0 && stride < (cols - 1) * ld + rows)
    return fail(ctx, LRB_ERR_SHAPE, "lrb_fill_uniform: stride %lld overlaps items", (long long)stride);
  if (batch == 0 || rows * cols == 0) return LRB_OK;
  if (!dst) return fail(ctx, LRB_ERR_ARG, "lrb_fill_uniform: dst is null");
  lrb_status st = lrb::bind(ctx);
  if (st) return st;
  const int64_t per = rows * cols;
  const unsigned bx = unsigned(std::min<int64_t>((per + 255) / 256, 64));
  const unsigned by = unsigned(std::min<int64_t>(batch, 65535));
  fill_strided_kernel<<<dim3(bx, by), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dst, rows, cols, ld, stride, batch, lrb_stream_key(seed, role), item_offset);
  LRB_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  return LRB_OK;
}

extern "C" lrb_status lrb_fill_uniform_ptr(lrb_ctx* ctx, double* const* dst, const int64_t* rows,
                                           const int64_t* cols, const int64_t* ld, int64_t batch,
                                           uint64_t seed, uint32_t role, int64_t item_offset,
                                           void* stream) {
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "lrb_fill_uniform_ptr: null ctx");
  if (batch < 0 || item_offset < 0) return fail(ctx, LRB_ERR_SHAPE, "lrb_fill_uniform_ptr: negative size");
  if (batch == 0) return LRB_OK;
  if (!dst || !rows || !cols || !ld) return fail(ctx, LRB_ERR_ARG, "lrb_fill_uniform_ptr: null array");
  std::vector<FillDesc> h(static_cast<size_t>(batch));
  for (int64_t i = 0; i < batch; ++i) {
    if (rows[i] < 0 || cols[i] < 0 || ld[i] < std::max<int64_t>(1, rows[i]))
      return fail(ctx, LRB_ERR_SHAPE, "lrb_fill_uniform_ptr: item %lld has a bad shape", (long long)i);
    if (rows[i] * cols[i] > 0 && !dst[i])
      return fail(ctx, LRB_ERR_ARG, "lrb_fill_uniform_ptr: item %lld dst is null", (long long)i);
    h[size_t(i)] = FillDesc{dst[i], rows[i], cols[i], ld[i]};
  }
  lrb_status st = lrb::bind(ctx);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FillDesc* d = nullptr;
  LRB_CUDA_TRY(ctx, lrb::pool_alloc(ctx, reinterpret_cast<void**>(&d), sizeof(FillDesc) * size_t(batch), s));
  LRB_CUDA_TRY(ctx, cudaMemcpyAsync(d, h.data(), sizeof(FillDesc) * size_t(batch),
                                    cudaMemcpyHostToDevice, s));
  const unsigned by = unsigned(std::min<int64_t>(batch, 65535));
  fill_ptr_kernel<<<dim3(64, by), 256, 0, s>>>(d, batch, lrb_stream_key(seed, role), item_offset);
  LRB_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  // h must outlive the async copy
  LRB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  LRB_CUDA_TRY(ctx, cudaFreeAsync(d, s));
  return LRB_OK;
}
