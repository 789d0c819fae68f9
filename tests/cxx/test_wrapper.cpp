// C++ host mirror (include/lrbatch_b200.hpp) through liblrb.so: the
// reference's known-answer tests (proj/tests/test_core.cpp:24-57) plus a
// batched device call checked bitwise against an in-order FMA chain.
// Exit 0 = all pass; prints one line per check.
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
  std::printf("%d failures\n", failures);
  return failures ? 1 : 0;
}
