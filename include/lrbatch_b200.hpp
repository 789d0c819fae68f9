// lrbatch_b200.hpp — C++ host layer over the C-ABI (include/lrb.h) that keeps
// the reference's contract for its hot path:
//
//   lrbatch::gemm_naive_raw(a, b, c, m, k, n, accumulate, flops)   dense.hpp:43-56
//   lrbatch::DenseBlock / dense_gemm_naive(...)                     dense.hpp:13-77
//   lrbatch::ShapeError / CapacityError / ParseError / IoError      common.hpp:19-37
//   lrbatch::LowRankBatch, flops_per_item                           low_rank.hpp:66-176
//   lrbatch::fused_multiply / packed_multiply / naive_multiply_batch
//                                                 kernels.hpp:131-349, bench.hpp:55-77
//   lrbatch::save_batch / load_batch                                batch_io.hpp:29-77
//   lrbatch::LowRankOperand, BlrMatrix, blr_matvec, reconstruct_dense  blr.hpp:15-202
//
// Same names, argument meaning and error behaviour (exceptions with the
// reference's messages, synchronous host-buffer calls, results overwritten or
// accumulated in place), computed on the B200 by liblrb.so. A reference user
// switches by including this header instead of <lrbatch/dense.hpp> and linking
// liblrb.so; the batched device-pointer entry points are added alongside.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <random>
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
class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& w) : std::runtime_error(w) {}
};
class IoError : public std::runtime_error {
 public:
  explicit IoError(const std::string& w) : std::runtime_error(w) {}
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
  if (st == LRB_ERR_PARSE) throw ParseError(msg);
  if (st == LRB_ERR_IO) throw IoError(msg);
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
  // variable-size batch over HOST blocks (the reference's own mode;
  // synchronous, copies pipelined with the kernels)
  void gemm_ptr_batched_host(char order, char opA, char opB, int64_t batch, const int64_t* m,
                             const int64_t* n, const int64_t* k, const double* const* A,
                             const int64_t* lda, const double* const* B, const int64_t* ldb,
                             double* const* C, const int64_t* ldc, bool accumulate) {
    check(lrb_dgemm_ptr_batched_host(h_, order, opA, opB, batch, m, n, k, A, lda, B, ldb, C, ldc,
                                     accumulate ? 1.0 : 0.0),
          h_);
  }
  // variable-size batch whose descriptor arrays live in DEVICE memory
  // (asynchronous; info: optional device int64_t[2])
  void gemm_ptr_batched_device(char order, char opA, char opB, int64_t batch, const int64_t* m,
                               const int64_t* n, const int64_t* k, const double* const* A,
                               const int64_t* lda, const double* const* B, const int64_t* ldb,
                               double* const* C, const int64_t* ldc, bool accumulate,
                               int64_t* info = nullptr, void* stream = nullptr) {
    check(lrb_dgemm_ptr_batched_device(h_, order, opA, opB, batch, m, n, k, A, lda, B, ldb, C,
                                       ldc, accumulate ? 1.0 : 0.0, info, stream),
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

// ===================================================== the low-rank product
// Seeded N(0, 1) source: std::mt19937_64 + std::normal_distribution, the
// standard-library generator the reference's NormalSource wraps
// (common.hpp:77-91), so random() batches equal the reference's.
class NormalSource {
 public:
  explicit NormalSource(std::uint64_t seed) : engine_(seed) {}
  double next() { return dist_(engine_); }
  void fill(double* dst, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) dst[i] = dist_(engine_);
  }

 private:
  std::mt19937_64 engine_;
  std::normal_distribution<double> dist_{0.0, 1.0};
};

// 4 r^3 + 2 r^2 b (low_rank.hpp:66-68)
inline std::uint64_t flops_per_item(std::uint64_t rank, std::uint64_t block_size) {
  return 4 * rank * rank * rank + 2 * rank * rank * block_size;
}

// Five role arrays, item i of a role at i * rows * cols, row-major
// (low_rank.hpp:109-176)
struct LowRankBatch {
  std::size_t batch_size = 0, block_size = 0, rank_a = 0, rank_b = 0;
  std::vector<double> a_vt_batch, b_u_batch, a_x_batch, b_x_batch, g_xy_batch;
  std::optional<std::uint64_t> seed;

  LowRankBatch() = default;
  LowRankBatch(std::size_t batch, std::size_t block, std::size_t ra, std::size_t rb)
      : batch_size(batch), block_size(block), rank_a(ra), rank_b(rb),
        a_vt_batch(batch * ra * block), b_u_batch(batch * block * rb), a_x_batch(batch * ra * ra),
        b_x_batch(batch * rb * rb), g_xy_batch(batch * ra * rb) {
    if (batch < 1) throw ShapeError("LowRankBatch: batch_size must be >= 1");
    if (block < 1) throw ShapeError("LowRankBatch: block_size must be >= 1");
    if (ra < 1 || rb < 1) throw ShapeError("LowRankBatch: ranks must be >= 1");
  }
  static LowRankBatch random(std::size_t batch, std::size_t block, std::size_t rank,
                             std::uint64_t seed) {
    LowRankBatch out(batch, block, rank, rank);
    NormalSource src(seed);
    src.fill(out.a_vt_batch.data(), out.a_vt_batch.size());
    src.fill(out.b_u_batch.data(), out.b_u_batch.size());
    src.fill(out.a_x_batch.data(), out.a_x_batch.size());
    src.fill(out.b_x_batch.data(), out.b_x_batch.size());
    out.seed = seed;
    return out;
  }
  const double* a_vt(std::size_t i) const { return a_vt_batch.data() + i * rank_a * block_size; }
  const double* b_u(std::size_t i) const { return b_u_batch.data() + i * block_size * rank_b; }
  const double* a_x(std::size_t i) const { return a_x_batch.data() + i * rank_a * rank_a; }
  const double* b_x(std::size_t i) const { return b_x_batch.data() + i * rank_b * rank_b; }
  double* g_xy(std::size_t i) { return g_xy_batch.data() + i * rank_a * rank_b; }
  const double* g_xy(std::size_t i) const { return g_xy_batch.data() + i * rank_a * rank_b; }
  void zero_results() { std::fill(g_xy_batch.begin(), g_xy_batch.end(), 0.0); }
  void validate() const {
    const std::size_t b = batch_size, k = block_size, ra = rank_a, rb = rank_b;
    if (!(b >= 1 && k >= 1 && ra >= 1 && rb >= 1))
      throw ShapeError("LowRankBatch: degenerate dimensions");
    if (a_vt_batch.size() != b * ra * k) throw ShapeError("LowRankBatch: a_vt_batch length mismatch");
    if (b_u_batch.size() != b * k * rb) throw ShapeError("LowRankBatch: b_u_batch length mismatch");
    if (a_x_batch.size() != b * ra * ra) throw ShapeError("LowRankBatch: a_x_batch length mismatch");
    if (b_x_batch.size() != b * rb * rb) throw ShapeError("LowRankBatch: b_x_batch length mismatch");
    if (g_xy_batch.size() != b * ra * rb) throw ShapeError("LowRankBatch: g_xy_batch length mismatch");
  }
};

// kernels.hpp:13-18; on the device only g_entry_stores is meaningful
struct MultiplyStats {
  std::uint64_t g_entry_stores = 0;
  double pack_small_seconds = 0.0;
  double pack_skinny_seconds = 0.0;
  double kernel_seconds = 0.0;
};

namespace detail {
inline void lowrank(LowRankBatch& batch, const char* who) {
  batch.validate();
  if (batch.rank_a != batch.rank_b)
    throw ShapeError(std::string(who) + ": rank_a must equal rank_b (got " +
                     std::to_string(batch.rank_a) + " and " + std::to_string(batch.rank_b) + ")");
  Context& ctx = default_context();
  check(lrb_lowrank_multiply_host(ctx.get(), int64_t(batch.batch_size), int64_t(batch.block_size),
                                  int64_t(batch.rank_a), batch.a_vt_batch.data(),
                                  batch.b_u_batch.data(), batch.a_x_batch.data(),
                                  batch.b_x_batch.data(), batch.g_xy_batch.data()),
        ctx.get());
}
}  // namespace detail

// fused_multiply (kernels.hpp:131-161) on the GPU
inline void fused_multiply(LowRankBatch& batch) { detail::lowrank(batch, "fused_multiply"); }

// packed_multiply (kernels.hpp:243-349) on the GPU: the CPU packing plan and
// worker count do not apply (any plan type is accepted and ignored)
template <class Plan>
inline void packed_multiply(LowRankBatch& batch, const Plan&, std::size_t = 1,
                            MultiplyStats* stats = nullptr) {
  detail::lowrank(batch, "packed_multiply");
  if (stats) stats->g_entry_stores += batch.batch_size * batch.rank_a * batch.rank_b;
}
inline void packed_multiply(LowRankBatch& batch) { detail::lowrank(batch, "packed_multiply"); }

// naive_multiply_batch (bench.hpp:55-77): the same device product
inline void naive_multiply_batch(LowRankBatch& batch, std::size_t = 1) {
  detail::lowrank(batch, "naive_multiply_batch");
}

// ------------------------------------------------------ LRBATCH1 batch files
inline void save_batch(const LowRankBatch& batch, const std::string& path) {
  batch.validate();
  check(lrb_batch_file_save(nullptr, path.c_str(), int64_t(batch.batch_size),
                            int64_t(batch.block_size), int64_t(batch.rank_a),
                            int64_t(batch.rank_b), batch.a_vt_batch.data(), batch.b_u_batch.data(),
                            batch.a_x_batch.data(), batch.b_x_batch.data(), 0),
        nullptr);
}

inline LowRankBatch load_batch(const std::string& path) {
  int64_t hdr[4] = {0, 0, 0, 0};
  check(lrb_batch_file_header(path.c_str(), hdr), nullptr);
  LowRankBatch out{static_cast<std::size_t>(hdr[0]), static_cast<std::size_t>(hdr[1]),
                   static_cast<std::size_t>(hdr[2]), static_cast<std::size_t>(hdr[3])};
  check(lrb_batch_file_load(nullptr, path.c_str(), out.a_vt_batch.data(), out.b_u_batch.data(),
                            out.a_x_batch.data(), out.b_x_batch.data(), 0),
        nullptr);
  return out;
}

// ============================================================ BLR matrices
// U (m x rank) X (rank x rank) Vt (rank x n), row-major (low_rank.hpp:16-63)
struct LowRankOperand {
  std::size_t m = 0, n = 0, rank = 0;
  std::vector<double> u, x, vt;

  LowRankOperand() = default;
  LowRankOperand(std::size_t m_, std::size_t n_, std::size_t r_)
      : m(m_), n(n_), rank(r_), u(m_ * r_), x(r_ * r_), vt(r_ * n_) {
    validate_dims();
  }
  LowRankOperand(std::size_t m_, std::size_t n_, std::size_t r_, std::vector<double> u_,
                 std::vector<double> x_, std::vector<double> vt_)
      : m(m_), n(n_), rank(r_), u(std::move(u_)), x(std::move(x_)), vt(std::move(vt_)) {
    validate_dims();
    if (u.size() != m * rank) throw ShapeError("LowRankOperand: u length != m*rank");
    if (x.size() != rank * rank) throw ShapeError("LowRankOperand: x length != rank*rank");
    if (vt.size() != rank * n) throw ShapeError("LowRankOperand: vt length != rank*n");
  }
  static LowRankOperand random(std::size_t m, std::size_t n, std::size_t rank, NormalSource& src) {
    LowRankOperand op(m, n, rank);
    src.fill(op.u.data(), op.u.size());
    src.fill(op.x.data(), op.x.size());
    src.fill(op.vt.data(), op.vt.size());
    return op;
  }
  std::size_t stored_entries() const { return m * rank + rank * rank + rank * n; }

 private:
  void validate_dims() const {
    if (rank < 1) throw ShapeError("LowRankOperand: rank must be >= 1");
    if (m < rank || n < rank)
      throw ShapeError("LowRankOperand: need m >= rank and n >= rank, got (" + std::to_string(m) +
                       ", " + std::to_string(n) + ", " + std::to_string(rank) + ")");
  }
};

// Weakly admissible BLR matrix (blr.hpp:15-87); the device copy is made on
// first use and kept until the tiles are edited (call invalidate())
struct BlrMatrix {
  std::size_t n = 0, block_size = 0, rank = 0, tiles = 0;
  std::vector<DenseBlock> diagonal;
  std::vector<LowRankOperand> off_diagonal;

  BlrMatrix(std::size_t n_, std::size_t block_, std::size_t rank_)
      : n(n_), block_size(block_), rank(rank_) {
    if (!(block_size >= 1 && n >= block_size)) throw ShapeError("BlrMatrix: bad block size");
    if (n % block_size != 0)
      throw ShapeError("BlrMatrix: n = " + std::to_string(n) +
                       " is not a multiple of block_size " + std::to_string(block_size));
    if (!(rank >= 1 && rank <= block_size))
      throw ShapeError("BlrMatrix: rank must be in [1, block]");
    tiles = n / block_size;
  }
  BlrMatrix(const BlrMatrix&) = delete;
  BlrMatrix& operator=(const BlrMatrix&) = delete;
  BlrMatrix(BlrMatrix&& o) noexcept { *this = std::move(o); }
  BlrMatrix& operator=(BlrMatrix&& o) noexcept {
    n = o.n, block_size = o.block_size, rank = o.rank, tiles = o.tiles;
    diagonal = std::move(o.diagonal);
    off_diagonal = std::move(o.off_diagonal);
    dev_ = o.dev_, dev_ctx_ = o.dev_ctx_;
    o.dev_ = nullptr, o.dev_ctx_ = nullptr;
    return *this;
  }
  ~BlrMatrix() { invalidate(); }

  std::size_t off_index(std::size_t i, std::size_t j) const {
    return i * (tiles - 1) + (j < i ? j : j - 1);
  }
  const LowRankOperand& off_tile(std::size_t i, std::size_t j) const {
    return off_diagonal[off_index(i, j)];
  }
  static BlrMatrix random(std::size_t n, std::size_t block, std::size_t rank, std::uint64_t seed) {
    BlrMatrix m(n, block, rank);
    NormalSource src(seed);
    for (std::size_t i = 0; i < m.tiles; ++i) {
      DenseBlock d(block, block);
      src.fill(d.data.data(), d.data.size());
      m.diagonal.push_back(std::move(d));
    }
    if (m.tiles > 1)
      for (std::size_t i = 0; i < m.tiles; ++i)
        for (std::size_t j = 0; j < m.tiles; ++j)
          if (i != j) m.off_diagonal.push_back(LowRankOperand::random(block, block, rank, src));
    return m;
  }
  void invalidate() {
    if (dev_) lrb_blr_destroy(dev_ctx_, dev_);
    dev_ = nullptr;
    dev_ctx_ = nullptr;
  }
  lrb_blr* device_handle(Context& ctx) const {
    if (dev_ && dev_ctx_ == ctx.get()) return dev_;
    const_cast<BlrMatrix*>(this)->invalidate();
    if (diagonal.size() != tiles || off_diagonal.size() != tiles * (tiles - 1))
      throw ShapeError("BlrMatrix: tiles are not populated");
    const std::size_t b = block_size, r = rank, T = tiles;
    std::vector<double> diag(T * b * b), u(T * (T - 1) * b * r + 1), x(T * (T - 1) * r * r + 1),
        vt(T * (T - 1) * r * b + 1);
    for (std::size_t i = 0; i < T; ++i)
      std::copy(diagonal[i].data.begin(), diagonal[i].data.end(), diag.begin() + i * b * b);
    for (std::size_t o = 0; o < off_diagonal.size(); ++o) {
      const LowRankOperand& t = off_diagonal[o];
      std::copy(t.u.begin(), t.u.end(), u.begin() + o * b * r);
      std::copy(t.x.begin(), t.x.end(), x.begin() + o * r * r);
      std::copy(t.vt.begin(), t.vt.end(), vt.begin() + o * r * b);
    }
    lrb_blr* h = nullptr;
    check(lrb_blr_create(ctx.get(), int64_t(n), int64_t(b), int64_t(r), diag.data(), u.data(),
                         x.data(), vt.data(), &h),
          ctx.get());
    dev_ = h;
    dev_ctx_ = ctx.get();
    return h;
  }
  // exact dense assembly (blr.hpp:62-86) on the GPU
  DenseBlock reconstruct_dense() const {
    Context& ctx = default_context();
    DenseBlock out(n, n);
    check(lrb_blr_reconstruct_dense(ctx.get(), device_handle(ctx), out.data.data(), 0, nullptr),
          ctx.get());
    return out;
  }

 private:
  mutable lrb_blr* dev_ = nullptr;
  mutable lrb_ctx* dev_ctx_ = nullptr;
};

// y = M rhs (blr_matvec, blr.hpp:141-175) on the GPU; plan/workers ignored
template <class Plan>
inline DenseBlock blr_matvec(const BlrMatrix& m, const DenseBlock& rhs, const Plan&,
                             std::size_t = 1) {
  if (rhs.rows != m.n)
    throw ShapeError("blr_matvec: rhs has " + std::to_string(rhs.rows) +
                     " rows, matrix has dimension " + std::to_string(m.n));
  Context& ctx = default_context();
  DenseBlock y(m.n, rhs.cols);
  check(lrb_blr_matvec(ctx.get(), m.device_handle(ctx), rhs.data.data(), int64_t(rhs.cols),
                       y.data.data()),
        ctx.get());
  return y;
}
inline DenseBlock blr_matvec(const BlrMatrix& m, const DenseBlock& rhs) {
  return blr_matvec(m, rhs, 0);
}
// blr_matvec_naive (blr.hpp:179-202): the same chain order, on the GPU
inline DenseBlock blr_matvec_naive(const BlrMatrix& m, const DenseBlock& rhs) {
  return blr_matvec(m, rhs, 0);
}

}  // namespace b200
}  // namespace lrbatch
