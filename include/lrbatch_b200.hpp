// lrbatch_b200.hpp — C++ host layer over the C-ABI (include/lrb.h) that keeps
// the reference's contract for its hot path:
//
//   lrbatch::gemm_naive_raw(a, b, c, m, k, n, accumulate, flops)   dense.hpp:43-56
//   lrbatch::DenseBlock / dense_gemm_naive(...)                     dense.hpp:13-77
//   lrbatch::ShapeError / CapacityError                             common.hpp:19-27
//
// Same names, argument meaning and error behaviour (exceptions with the
// reference's messages, synchronous host-buffer calls, results overwritten or
// accumulated in place), computed on the B200 by liblrb.so. A reference user
// switches by including this header instead of <lrbatch/dense.hpp> and linking
// liblrb.so; the batched device-pointer entry points are added alongside.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lrb.h"

namespace lrbatch {
namespace b200 {

class ShapeError : public std::invalid_argument {
 public:
  explicit ShapeError(const std::string& w) : std::invalid_argument(w) {}
};
class CapacityError : public std::runtime_error {
 public:
  explicit CapacityError(const std::string& w) : std::runtime_error(w) {}
};
class DeviceError : public std::runtime_error {
 public:
  DeviceError(lrb_status s, const std::string& w) : std::runtime_error(w), status(s) {}
  lrb_status status;
};

inline void check(lrb_status st, const lrb_ctx* ctx) {
  if (st == LRB_OK) return;
  const char* m = lrb_last_error(ctx);
  std::string msg = m ? m : "lrb error";
  if (st == LRB_ERR_SHAPE) throw ShapeError(msg);
  if (st == LRB_ERR_CAPACITY) throw CapacityError(msg);
  throw DeviceError(st, msg);
}

// RAII owner of one lrb_ctx (one per host thread and device)
class Context {
 public:
  explicit Context(int device = 0) { check(lrb_create(device, &h_), nullptr); }
  ~Context() { lrb_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lrb_ctx* get() const { return h_; }
  int device() const { return lrb_ctx_device(h_); }
  uint64_t launch_count() const { return lrb_launch_count(h_); }

  // column-major (order 'C') or row-major ('R') strided batch on DEVICE pointers
  void gemm_strided_batched(char order, char opA, char opB, int64_t m, int64_t n, int64_t k,
                            bool accumulate, const double* A, int64_t lda, int64_t strideA,
                            const double* B, int64_t ldb, int64_t strideB, double* C,
                            int64_t ldc, int64_t strideC, int64_t batch, void* stream = nullptr) {
    check(lrb_dgemm_strided_batched(h_, order, opA, opB, m, n, k, accumulate ? 1.0 : 0.0, A, lda,
                                    strideA, B, ldb, strideB, C, ldc, strideC, batch, stream),
          h_);
  }
  // the same on HOST buffers (synchronous; H2D / kernel / D2H pipelined)
  void gemm_strided_batched_host(char order, char opA, char opB, int64_t m, int64_t n, int64_t k,
                                 bool accumulate, const double* A, int64_t lda, int64_t strideA,
                                 const double* B, int64_t ldb, int64_t strideB, double* C,
                                 int64_t ldc, int64_t strideC, int64_t batch) {
    check(lrb_dgemm_strided_batched_host(h_, order, opA, opB, m, n, k, accumulate ? 1.0 : 0.0, A,
                                         lda, strideA, B, ldb, strideB, C, ldc, strideC, batch),
          h_);
  }
  void synchronize() { check(lrb_device_sync(h_), h_); }

 private:
  lrb_ctx* h_ = nullptr;
};

// the calling thread's context on device 0, created on first use
inline Context& default_context() {
  thread_local std::unique_ptr<Context> ctx;
  if (!ctx) ctx.reset(new Context(0));
  return *ctx;
}

// Drop-in for lrbatch::gemm_naive_raw (dense.hpp:43-56): row-major host
// buffers, c = [c] + a * b, flops += 2*m*n*k when non-null.
inline void gemm_naive_raw(const double* a, const double* b, double* c, std::size_t m,
                           std::size_t k, std::size_t n, bool accumulate,
                           std::uint64_t* flops = nullptr) {
  Context& ctx = default_context();
  check(lrb_gemm_naive_raw(ctx.get(), a, b, c, m, k, n, accumulate ? 1 : 0, flops), ctx.get());
}

// Row-major dense block (reference DenseBlock, dense.hpp:13-37)
struct DenseBlock {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<double> data;

  DenseBlock() = default;
  DenseBlock(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
  DenseBlock(std::size_t r, std::size_t c, std::vector<double> d)
      : rows(r), cols(c), data(std::move(d)) {
    if (data.size() != rows * cols)
      throw ShapeError("DenseBlock: data length " + std::to_string(data.size()) +
                       " != rows*cols " + std::to_string(rows * cols));
  }
  double& at(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  double at(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
  static DenseBlock identity(std::size_t n) {
    DenseBlock b(n, n);
    for (std::size_t i = 0; i < n; ++i) b.at(i, i) = 1.0;
    return b;
  }
};

// dense_gemm_naive (dense.hpp:58-77): same checks, same messages
inline void dense_gemm_naive(const DenseBlock& a, const DenseBlock& b, DenseBlock& out,
                             bool accumulate, std::uint64_t* flops = nullptr) {
  if (a.cols != b.rows)
    throw ShapeError("dense_gemm_naive: a is " + std::to_string(a.rows) + "x" +
                     std::to_string(a.cols) + " but b is " + std::to_string(b.rows) + "x" +
                     std::to_string(b.cols));
  if (out.rows != a.rows || out.cols != b.cols)
    throw ShapeError("dense_gemm_naive: output is " + std::to_string(out.rows) + "x" +
                     std::to_string(out.cols) + ", expected " + std::to_string(a.rows) + "x" +
                     std::to_string(b.cols));
  gemm_naive_raw(a.data.data(), b.data.data(), out.data.data(), a.rows, a.cols, b.cols,
                 accumulate, flops);
}

inline DenseBlock dense_gemm_naive(const DenseBlock& a, const DenseBlock& b,
                                   std::uint64_t* flops = nullptr) {
  DenseBlock out(a.rows, b.cols);
  dense_gemm_naive(a, b, out, false, flops);
  return out;
}

}  // namespace b200
}  // namespace lrbatch
