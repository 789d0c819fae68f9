// C++ host mirror (include/lrbatch_b200.hpp) through liblrb.so: the
// reference's known-answer tests (proj/tests/test_core.cpp:24-57) plus a
// batched device call checked bitwise against an in-order FMA chain.
// Exit 0 = all pass; prints one line per check.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "lrbatch_b200.hpp"

using namespace lrbatch::b200;

static int failures = 0;
#define CHECK(cond, name)                                   \
  do {                                                      \
    bool ok_ = (cond);                                      \
    std::printf("%s %s\n", ok_ ? "PASS" : "FAIL", name);    \
    if (!ok_) ++failures;                                   \
  } while (0)

int main() {
  // known answers (test_core.cpp:24-39)
  DenseBlock id = DenseBlock::identity(3);
  DenseBlock m(3, 3, {1, 2, 3, 4, 5, 6, 7, 8, 9});
  CHECK(dense_gemm_naive(id, m).data == m.data, "identity * M == M");
  DenseBlock z(2, 5), any(5, 4, std::vector<double>(20, 3.25));
  DenseBlock zr = dense_gemm_naive(z, any);
  bool allz = true;
  for (double v : zr.data) allz = allz && v == 0.0;
  CHECK(allz, "zeros * X == 0");
  DenseBlock a(2, 2, {1, 2, 3, 4}), b(2, 2, {5, 6, 7, 8});
  CHECK((dense_gemm_naive(a, b).data == std::vector<double>{19, 22, 43, 50}), "2x2 product");
  // accumulate flag (test_core.cpp:41-49)
  DenseBlock e(2, 2, {1, 0, 0, 1}), f(2, 2, {1, 2, 3, 4}), out(2, 2, {10, 10, 10, 10});
  dense_gemm_naive(e, f, out, true);
  CHECK((out.data == std::vector<double>{11, 12, 13, 14}), "accumulate");
  dense_gemm_naive(e, f, out, false);
  CHECK(out.data == f.data, "overwrite");
  // shape error names both shapes (test_core.cpp:51-57)
  bool threw = false;
  try {
    DenseBlock p(2, 3), q(4, 2);
    dense_gemm_naive(p, q);
  } catch (const ShapeError& ex) {
    std::string w = ex.what();
    threw = w.find("2x3") != std::string::npos && w.find("4x2") != std::string::npos;
  }
  CHECK(threw, "ShapeError names 2x3 and 4x2");
  // flops counter
  std::uint64_t fl = 7;
  std::vector<double> x(6 * 5, 1.0), y(5 * 4, 2.0), r(6 * 4, 0.0);
  gemm_naive_raw(x.data(), y.data(), r.data(), 6, 5, 4, false, &fl);
  CHECK(fl == 7 + 2 * 6 * 5 * 4 && r[0] == 10.0, "flops counter and values");

  // batched, column-major, host buffers: bitwise vs the in-order FMA chain
  const int M = 129, N = 23, K = 77, BATCH = 5;
  std::mt19937_64 gen(42);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> A(M * K * BATCH), B(K * N * BATCH), C(M * N * BATCH, NAN), W(M * N * BATCH);
  for (auto& v : A) v = U(gen);
  for (auto& v : B) v = U(gen);
  Context& ctx = default_context();
  ctx.gemm_strided_batched_host('C', 'N', 'N', M, N, K, false, A.data(), M, M * K, B.data(), K,
                                K * N, C.data(), M, M * N, BATCH);
  for (int it = 0; it < BATCH; ++it)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < M; ++i) {
        double s = 0.0;
        for (int p = 0; p < K; ++p)
          s = std::fma(A[it * M * K + i + p * M], B[it * K * N + p + j * K], s);
        W[it * M * N + i + j * M] = s;
      }
  CHECK(C == W, "batched column-major == FMA chain (bitwise)");
  CHECK(ctx.launch_count() > 0, "kernels launched");
  // bad leading dimension -> ShapeError
  threw = false;
  try {
    ctx.gemm_strided_batched_host('C', 'N', 'N', M, N, K, false, A.data(), M - 1, M * K, B.data(),
                                  K, K * N, C.data(), M, M * N, BATCH);
  } catch (const ShapeError&) {
    threw = true;
  }
  CHECK(threw, "lda < m raises ShapeError");

  // variable-size pointer-array batch over host blocks (cfg4's shape family)
  {
    const int64_t nb = 4;
    const int64_t bm[nb] = {256, 512, 256, 130}, rn[nb] = {8, 37, 64, 13};
    std::vector<std::vector<double>> a(nb), b(nb), c(nb), w(nb);
    std::vector<const double*> pa(nb), pb(nb);
    std::vector<double*> pc(nb);
    for (int64_t i = 0; i < nb; ++i) {
      a[i].resize(bm[i] * bm[i]);
      b[i].resize(bm[i] * rn[i]);
      c[i].assign(bm[i] * rn[i], NAN);
      w[i].resize(bm[i] * rn[i]);
      for (auto& v : a[i]) v = U(gen);
      for (auto& v : b[i]) v = U(gen);
      pa[i] = a[i].data();
      pb[i] = b[i].data();
      pc[i] = c[i].data();
      for (int64_t j = 0; j < rn[i]; ++j)
        for (int64_t r = 0; r < bm[i]; ++r) {
          double s = 0.0;
          for (int64_t p = 0; p < bm[i]; ++p) s = std::fma(a[i][r + p * bm[i]], b[i][p + j * bm[i]], s);
          w[i][r + j * bm[i]] = s;
        }
    }
    ctx.gemm_ptr_batched_host('C', 'N', 'N', nb, bm, rn, bm, pa.data(), bm, pb.data(), bm,
                              pc.data(), bm, false);
    bool same = true;
    for (int64_t i = 0; i < nb; ++i) same = same && c[i] == w[i];
    CHECK(same, "pointer-array host batch == FMA chain (bitwise)");
  }

  // ------------------------------------------------- the low-rank product
  // all-ones factors (test_core.cpp:59-67): block 1 -> 1, block 4 -> 4
  {
    LowRankBatch one(1, 1, 1, 1), four(1, 4, 1, 1);
    for (LowRankBatch* b : {&one, &four}) {
      std::fill(b->a_vt_batch.begin(), b->a_vt_batch.end(), 1.0);
      std::fill(b->b_u_batch.begin(), b->b_u_batch.end(), 1.0);
      std::fill(b->a_x_batch.begin(), b->a_x_batch.end(), 1.0);
      std::fill(b->b_x_batch.begin(), b->b_x_batch.end(), 1.0);
    }
    fused_multiply(one);
    packed_multiply(four);
    CHECK(one.g_xy_batch[0] == 1.0 && four.g_xy_batch[0] == 4.0, "all-ones low-rank product");
  }
  // random batch: G = A_X (A_Vt B_U) B_X bitwise vs three FMA chains
  {
    const std::size_t n = 9, blk = 256, r = 16;
    LowRankBatch lb = LowRankBatch::random(n, blk, r, 7);
    MultiplyStats stats;
    packed_multiply(lb, /*plan=*/0, 4, &stats);
    bool same = true;
    std::vector<double> c(r * r), e(r * r);
    for (std::size_t it = 0; it < n; ++it) {
      const double *av = lb.a_vt(it), *bu = lb.b_u(it), *ax = lb.a_x(it), *bx = lb.b_x(it);
      for (std::size_t i = 0; i < r; ++i)
        for (std::size_t j = 0; j < r; ++j) {
          double s = 0.0;
          for (std::size_t p = 0; p < blk; ++p) s = std::fma(av[i * blk + p], bu[p * r + j], s);
          c[i * r + j] = s;
        }
      for (std::size_t i = 0; i < r; ++i)
        for (std::size_t j = 0; j < r; ++j) {
          double s = 0.0;
          for (std::size_t p = 0; p < r; ++p) s = std::fma(ax[i * r + p], c[p * r + j], s);
          e[i * r + j] = s;
        }
      for (std::size_t i = 0; i < r; ++i)
        for (std::size_t j = 0; j < r; ++j) {
          double s = 0.0;
          for (std::size_t p = 0; p < r; ++p) s = std::fma(e[i * r + p], bx[p * r + j], s);
          same = same && s == lb.g_xy(it)[i * r + j];
        }
    }
    CHECK(same, "packed_multiply == FMA-chain product (bitwise)");
    CHECK(stats.g_entry_stores == n * r * r, "g_entry_stores");
    LowRankBatch again = LowRankBatch::random(n, blk, r, 7);
    naive_multiply_batch(again, 3);
    CHECK(again.g_xy_batch == lb.g_xy_batch, "naive_multiply_batch == packed_multiply");
  }
  threw = false;
  try {
    LowRankBatch bad(2, 16, 4, 8);
    fused_multiply(bad);
  } catch (const ShapeError& ex) {
    threw = std::string(ex.what()).find("rank_a must equal rank_b") != std::string::npos;
  }
  CHECK(threw, "rank mismatch raises ShapeError");

  // ------------------------------------------------------ LRBATCH1 files
  {
    LowRankBatch lb = LowRankBatch::random(5, 32, 4, 11);
    const std::string path = "/tmp/lrb_cxx_test.lrb";
    save_batch(lb, path);
    LowRankBatch back = load_batch(path);
    CHECK(back.batch_size == 5 && back.block_size == 32 && back.rank_a == 4 &&
              back.a_vt_batch == lb.a_vt_batch && back.b_x_batch == lb.b_x_batch,
          "save_batch / load_batch round trip");
    bool io = false, parse = false;
    try {
      load_batch("/tmp/definitely/not/here.lrb");
    } catch (const IoError&) {
      io = true;
    }
    {
      FILE* f = std::fopen(path.c_str(), "wb");
      std::fputs("NOTABATCHFILE...", f);
      std::fclose(f);
    }
    try {
      load_batch(path);
    } catch (const ParseError&) {
      parse = true;
    }
    std::remove(path.c_str());
    CHECK(io && parse, "IoError / ParseError");
  }

  // ---------------------------------------------------------- BLR matvec
  {
    BlrMatrix m = BlrMatrix::random(192, 32, 6, 5);
    DenseBlock rhs(192, 3);
    NormalSource src(9);
    src.fill(rhs.data.data(), rhs.data.size());
    DenseBlock y = blr_matvec(m, rhs, /*plan=*/0, 2);
    DenseBlock expect = dense_gemm_naive(m.reconstruct_dense(), rhs);
    double rms = 0.0;
    for (double v : expect.data) rms += v * v;
    rms = std::sqrt(rms / double(expect.data.size()));
    double worst = 0.0;
    for (std::size_t i = 0; i < y.data.size(); ++i)
      worst = std::max(worst, std::fabs(y.data[i] - expect.data[i]) /
                                  std::max(std::fabs(expect.data[i]), rms));
    CHECK(worst < 1e-10, "blr_matvec == reconstruct_dense * rhs");
    CHECK(blr_matvec_naive(m, rhs).data == y.data, "blr_matvec_naive == blr_matvec");
    bool shape = false;
    try {
      blr_matvec(m, DenseBlock(100, 2));
    } catch (const ShapeError&) {
      shape = true;
    }
    CHECK(shape, "rhs row mismatch raises ShapeError");
  }
  std::printf("%d failures\n", failures);
  return failures ? 1 : 0;
}
