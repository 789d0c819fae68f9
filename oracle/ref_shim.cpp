// ref_shim.cpp — builds the UNMODIFIED reference oracle into oracle/_ref/.
//
// TEST INFRASTRUCTURE ONLY: the reference itself, compiled from its own header
// (/root/reference/proj/include/lrbatch/dense.hpp) by the top-level Makefile's
// `ref` target, to pin the C restatement (oracle/lrb_oracle.c), to generate
// the golden vectors under tests/golden/, and as the CPU baseline
// (`cpu_baseline.kind = "reference"`, `bench.py --impl reference`). No
// reference source is copied into this repository; this file only includes it.
#include <lrbatch/dense.hpp>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <type_traits>
#include <vector>

namespace {

bool is_t(char o) { return o == 'T' || o == 't'; }

// One column-major item through the reference primitive: the
// column-major product C = op(A) op(B) has the bytes of the row-major
// C^T = op(B)^T op(A)^T, so the reference is called as
// gemm_naive_raw(op(B)^T, op(A)^T, C^T, n, k, m, accumulate) with operand
// copies only where the stored layout is not already that row-major one
// (transposes, padded leading dimensions). Per-entry order is unchanged.
void colmajor_item(char opA, char opB, int64_t m, int64_t n, int64_t k, bool acc, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                   std::vector<double>& sa, std::vector<double>& sb, std::vector<double>& sc) {
  // a' = op(B)^T as row-major n x k: a'[j*k + p] = op(B)(p, j)
  const double* ap;
  if (!is_t(opB) && ldb == k) {
    ap = B;  // column-major k x n with ld k == row-major n x k
  } else {
    sa.resize(size_t(n * k));
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = 0; p < k; ++p)
        sa[size_t(j * k + p)] = is_t(opB) ? B[j + p * ldb] : B[p + j * ldb];
    ap = sa.data();
  }
  // b' = op(A)^T as row-major k x m: b'[p*m + i] = op(A)(i, p)
  const double* bp;
  if (!is_t(opA) && lda == m) {
    bp = A;
  } else {
    sb.resize(size_t(k * m));
    for (int64_t p = 0; p < k; ++p)
      for (int64_t i = 0; i < m; ++i)
        sb[size_t(p * m + i)] = is_t(opA) ? A[p + i * lda] : A[i + p * lda];
    bp = sb.data();
  }
  if (ldc == m) {
    lrbatch::gemm_naive_raw(ap, bp, C, size_t(n), size_t(k), size_t(m), acc);
  } else {
    sc.assign(size_t(n * m), 0.0);
    if (acc)
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) sc[size_t(j * m + i)] = C[i + j * ldc];
    lrbatch::gemm_naive_raw(ap, bp, sc.data(), size_t(n), size_t(k), size_t(m), acc);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) C[i + j * ldc] = sc[size_t(j * m + i)];
  }
}

template <class Body>
void fan_out(int64_t batch, int threads, Body body) {
  // contiguous split, as naive_multiply_batch (reference bench.hpp:59-76)
  int64_t workers = std::max<int64_t>(1, std::min<int64_t>(threads, batch));
  if (workers == 1) {
    body(int64_t(0), batch);
    return;
  }
  const int64_t per = (batch + workers - 1) / workers;
  std::vector<std::thread> pool;
  for (int64_t w = 1; w < workers; ++w) {
    const int64_t b = std::min(w * per, batch), e = std::min(b + per, batch);
    pool.emplace_back(body, b, e);
  }
  body(int64_t(0), std::min(per, batch));
  for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

// the reference primitive itself
void ref_gemm_naive_raw(const double* a, const double* b, double* c, size_t m, size_t k, size_t n,
                        int accumulate, uint64_t* flops) {
  lrbatch::gemm_naive_raw(a, b, c, m, k, n, accumulate != 0, flops);
}

// row-major strided batch exactly as the reference packs LowRankBatch roles
// (low_rank.hpp:147-158): one gemm_naive_raw per item
void ref_gemm_rowmajor_batched(const double* a, const double* b, double* c, size_t m, size_t k,
                               size_t n, int accumulate, int64_t batch, int threads) {
  fan_out(batch, threads, [&](int64_t b0, int64_t e0) {
    for (int64_t it = b0; it < e0; ++it)
      lrbatch::gemm_naive_raw(a + it * m * k, b + it * k * n, c + it * m * n, m, k, n,
                              accumulate != 0);
  });
}

// column-major strided batch through the reference primitive (operand swap)
int ref_dgemm_colmajor_strided(char opA, char opB, int64_t m, int64_t n, int64_t k, int accumulate,
                               const double* A, int64_t lda, int64_t sA, const double* B,
                               int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC,
                               int64_t batch, int threads) {
  if (m < 0 || n < 0 || k < 0 || batch < 0) return -1;
  fan_out(batch, threads, [&](int64_t b0, int64_t e0) {
    std::vector<double> sa, sb, sc;
    for (int64_t it = b0; it < e0; ++it)
      colmajor_item(opA, opB, m, n, k, accumulate != 0, A + it * sA, lda, B + it * sB, ldb,
                    C + it * sC, ldc, sa, sb, sc);
  });
  return 0;
}

// column-major pointer-array batch through the reference primitive
int ref_dgemm_colmajor_ptr(char opA, char opB, int64_t batch, const int64_t* m, const int64_t* n,
                           const int64_t* k, const double* const* A, const int64_t* lda,
                           const double* const* B, const int64_t* ldb, double* const* C,
                           const int64_t* ldc, int accumulate, int threads) {
  fan_out(batch, threads, [&](int64_t b0, int64_t e0) {
    std::vector<double> sa, sb, sc;
    for (int64_t it = b0; it < e0; ++it)
      colmajor_item(opA, opB, m[it], n[it], k[it], accumulate != 0, A[it], lda[it], B[it], ldb[it],
                    C[it], ldc[it], sa, sb, sc);
  });
  return 0;
}

// dense_gemm_naive's ShapeError text for shapes (ar x ac) * (br x bc) with an
// (or x oc) output; returns 1 and fills buf when it throws, else 0
int ref_dense_gemm_naive_error(size_t ar, size_t ac, size_t br, size_t bc, size_t orow, size_t ocol,
                               char* buf, size_t buflen) {
  try {
    lrbatch::DenseBlock a(ar, ac), b(br, bc), out(orow, ocol);
    lrbatch::dense_gemm_naive(a, b, out, false);
  } catch (const lrbatch::ShapeError& e) {
    std::strncpy(buf, e.what(), buflen - 1);
    buf[buflen - 1] = 0;
    return 1;
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The paper's batched low-rank product through the reference's own drivers.
#include <lrbatch/bench.hpp>
#include <lrbatch/kernels.hpp>
#include <lrbatch/machine.hpp>
#include <lrbatch/verify.hpp>

namespace {
// wall time of the last reference driver call alone (no marshalling into the
// reference's containers), read back with ref_last_seconds()
double g_last_seconds = 0.0;

template <class F>
auto timed(F&& f) {
  const auto t0 = std::chrono::steady_clock::now();
  auto finish = [&] {
    g_last_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  if constexpr (std::is_void_v<decltype(f())>) {
    f();
    finish();
  } else {
    auto r = f();
    finish();
    return r;
  }
}

// PackingPlan <-> 10 int64 fields (plan.hpp:21-31), so a plan the reference
// derived here from its machine files can be replayed where they are absent
constexpr int kPlanFields = 10;

void plan_to_fields(const lrbatch::PackingPlan& p, int64_t* f) {
  f[0] = int64_t(p.b_small);
  f[1] = int64_t(p.b_skinny);
  f[2] = int64_t(p.m_pack);
  f[3] = int64_t(p.n_pack);
  f[4] = int64_t(p.x_pack);
  f[5] = int64_t(p.y_pack);
  f[6] = int64_t(p.tile);
  f[7] = int64_t(p.llc_bytes);
  f[8] = int64_t(p.alignment_bytes);
  f[9] = p.dual_accumulator ? 1 : 0;
}

lrbatch::PackingPlan plan_from(const int64_t* f, const char* machine, size_t rank, size_t block) {
  if (!f)
    return lrbatch::make_packing_plan(lrbatch::resolve_machine(machine ? machine : "skylake-x-6148"),
                                      rank, block);
  lrbatch::PackingPlan p;
  p.b_small = size_t(f[0]);
  p.b_skinny = size_t(f[1]);
  p.m_pack = size_t(f[2]);
  p.n_pack = size_t(f[3]);
  p.x_pack = size_t(f[4]);
  p.y_pack = size_t(f[5]);
  p.tile = size_t(f[6]);
  p.llc_bytes = size_t(f[7]);
  p.alignment_bytes = size_t(f[8]);
  p.dual_accumulator = f[9] != 0;
  return p;
}

lrbatch::LowRankBatch make_batch(int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                                 const double* b_u, const double* a_x, const double* b_x) {
  lrbatch::LowRankBatch lb{size_t(batch), size_t(block), size_t(rank), size_t(rank)};
  std::memcpy(lb.a_vt_batch.data(), a_vt, sizeof(double) * lb.a_vt_batch.size());
  std::memcpy(lb.b_u_batch.data(), b_u, sizeof(double) * lb.b_u_batch.size());
  std::memcpy(lb.a_x_batch.data(), a_x, sizeof(double) * lb.a_x_batch.size());
  std::memcpy(lb.b_x_batch.data(), b_x, sizeof(double) * lb.b_x_batch.size());
  return lb;
}
}  // namespace

extern "C" {

double ref_last_seconds() { return g_last_seconds; }

// make_packing_plan (plan.hpp:66-100) for `machine` -> 10 fields; 0 on success
int ref_packing_plan(const char* machine, int64_t rank, int64_t block, int64_t* fields) {
  try {
    plan_to_fields(plan_from(nullptr, machine, size_t(rank), size_t(block)), fields);
  } catch (...) {
    return -1;
  }
  return 0;
}

// which: 0 naive_multiply_batch (the reference CPU baseline, bench.hpp:55-77),
//        1 fused_multiply (kernels.hpp:131-161),
//        2 packed_multiply (kernels.hpp:243-349) with `plan` (10 fields) or,
//          when plan is NULL, make_packing_plan for `machine`
int ref_lowrank_multiply(int which, int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                         const double* b_u, const double* a_x, const double* b_x, double* g,
                         int workers, const char* machine, const int64_t* plan) {
  try {
    lrbatch::LowRankBatch lb = make_batch(batch, block, rank, a_vt, b_u, a_x, b_x);
    if (which == 0) {
      timed([&] { lrbatch::naive_multiply_batch(lb, size_t(workers)); });
    } else if (which == 1) {
      timed([&] { lrbatch::fused_multiply(lb); });
    } else {
      const lrbatch::PackingPlan pp = plan_from(plan, machine, size_t(rank), size_t(block));
      timed([&] { lrbatch::packed_multiply(lb, pp, size_t(workers)); });
    }
    std::memcpy(g, lb.g_xy_batch.data(), sizeof(double) * lb.g_xy_batch.size());
  } catch (...) {
    return -1;
  }
  return 0;
}

// compare_to_reference (verify.hpp:38-64) of `g` against the reference oracle
double ref_compare_to_reference(int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                                const double* b_u, const double* a_x, const double* b_x,
                                const double* g, int64_t* worst_item, int64_t* worst_entry) {
  lrbatch::LowRankBatch lb = make_batch(batch, block, rank, a_vt, b_u, a_x, b_x);
  std::memcpy(lb.g_xy_batch.data(), g, sizeof(double) * lb.g_xy_batch.size());
  lrbatch::VerifyReport rep = lrbatch::compare_to_reference(lb, 1.0);
  if (worst_item) *worst_item = int64_t(rep.worst_item);
  if (worst_entry) *worst_entry = int64_t(rep.worst_entry);
  return rep.max_rel_error;
}

}  // extern "C"

#include <lrbatch/batch_io.hpp>

extern "C" {
// the reference's own save_batch / load_batch (batch_io.hpp:29-77)
int ref_save_batch(const char* path, int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                   const double* b_u, const double* a_x, const double* b_x) {
  try {
    lrbatch::save_batch(make_batch(batch, block, rank, a_vt, b_u, a_x, b_x), path);
  } catch (...) {
    return -1;
  }
  return 0;
}

// returns 0 and the arrays, or 1 + the exception text in `err`
int ref_load_batch(const char* path, int64_t* hdr, double* a_vt, double* b_u, double* a_x,
                   double* b_x, char* err, size_t errlen) {
  try {
    lrbatch::LowRankBatch lb = lrbatch::load_batch(path);
    hdr[0] = int64_t(lb.batch_size);
    hdr[1] = int64_t(lb.block_size);
    hdr[2] = int64_t(lb.rank_a);
    hdr[3] = int64_t(lb.rank_b);
    if (a_vt) std::memcpy(a_vt, lb.a_vt_batch.data(), lb.a_vt_batch.size() * 8);
    if (b_u) std::memcpy(b_u, lb.b_u_batch.data(), lb.b_u_batch.size() * 8);
    if (a_x) std::memcpy(a_x, lb.a_x_batch.data(), lb.a_x_batch.size() * 8);
    if (b_x) std::memcpy(b_x, lb.b_x_batch.data(), lb.b_x_batch.size() * 8);
  } catch (const std::exception& e) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
    return 1;
  }
  return 0;
}
}  // extern "C"

#include <lrbatch/blr.hpp>

extern "C" {
// which: 0 blr_matvec (packed path; `plan` fields, or the plan for `machine`
// at rank max(rank, nrhs) when NULL), 1 blr_matvec_naive,
// 2 dense_gemm_naive(reconstruct_dense(), rhs) — blr.hpp:64-202
int ref_blr_matvec(int which, int64_t n, int64_t block, int64_t rank, const double* diag,
                   const double* u, const double* x, const double* vt, const double* rhs,
                   int64_t nrhs, double* y, int workers, const char* machine,
                   const int64_t* plan) {
  try {
    lrbatch::BlrMatrix m{size_t(n), size_t(block), size_t(rank)};
    const size_t T = m.tiles, b = size_t(block), r = size_t(rank);
    for (size_t i = 0; i < T; ++i)
      m.diagonal.emplace_back(b, b, std::vector<double>(diag + i * b * b, diag + (i + 1) * b * b));
    for (size_t o = 0; o < T * (T - 1); ++o)
      m.off_diagonal.emplace_back(b, b, r, std::vector<double>(u + o * b * r, u + (o + 1) * b * r),
                                  std::vector<double>(x + o * r * r, x + (o + 1) * r * r),
                                  std::vector<double>(vt + o * r * b, vt + (o + 1) * r * b));
    lrbatch::DenseBlock rb{size_t(n), size_t(nrhs),
                           std::vector<double>(rhs, rhs + size_t(n) * size_t(nrhs))};
    lrbatch::DenseBlock out;
    if (which == 0) {
      const lrbatch::PackingPlan pp = plan_from(plan, machine, std::max(r, size_t(nrhs)), b);
      out = timed([&] { return lrbatch::blr_matvec(m, rb, pp, size_t(workers)); });
    } else if (which == 1) {
      out = timed([&] { return lrbatch::blr_matvec_naive(m, rb); });
    } else {
      const lrbatch::DenseBlock dense = m.reconstruct_dense();
      out = timed([&] { return lrbatch::dense_gemm_naive(dense, rb); });
    }
    std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
  } catch (...) {
    return -1;
  }
  return 0;
}
}  // extern "C"

extern "C" {
// BlrMatrix::reconstruct_dense (blr.hpp:62-86) -> out (n x n, row-major)
int ref_blr_reconstruct(int64_t n, int64_t block, int64_t rank, const double* diag,
                        const double* u, const double* x, const double* vt, double* out) {
  try {
    lrbatch::BlrMatrix m{size_t(n), size_t(block), size_t(rank)};
    const size_t T = m.tiles, b = size_t(block), r = size_t(rank);
    for (size_t i = 0; i < T; ++i)
      m.diagonal.emplace_back(b, b, std::vector<double>(diag + i * b * b, diag + (i + 1) * b * b));
    for (size_t o = 0; o < T * (T - 1); ++o)
      m.off_diagonal.emplace_back(b, b, r, std::vector<double>(u + o * b * r, u + (o + 1) * b * r),
                                  std::vector<double>(x + o * r * r, x + (o + 1) * r * r),
                                  std::vector<double>(vt + o * r * b, vt + (o + 1) * r * b));
    const lrbatch::DenseBlock full = timed([&] { return m.reconstruct_dense(); });
    std::memcpy(out, full.data.data(), full.data.size() * sizeof(double));
  } catch (...) {
    return -1;
  }
  return 0;
}

// the per-tile expansion of reconstruct_dense (blr.hpp:75-78) over a batch of
// contiguous LowRankOperands: out_i = (U_i X_i) Vt_i through the reference's
// gemm_naive_raw (what dense_gemm_naive runs after its shape checks,
// dense.hpp:58-77), items split over `workers` threads like
// naive_multiply_batch; ref_last_seconds() covers the products alone.
int ref_lowrank_expand(int64_t batch, int64_t m, int64_t n, int64_t rank, const double* u,
                       const double* x, const double* vt, double* out, int workers) {
  if (batch < 0 || m < 1 || n < 1 || rank < 1) return -1;
  const size_t M = size_t(m), N = size_t(n), R = size_t(rank);
  timed([&] {
    fan_out(batch, workers, [&](int64_t b0, int64_t e0) {
      std::vector<double> ux(M * R);
      for (int64_t it = b0; it < e0; ++it) {
        lrbatch::gemm_naive_raw(u + it * M * R, x + it * R * R, ux.data(), M, R, R, false);
        lrbatch::gemm_naive_raw(ux.data(), vt + it * R * N, out + it * M * N, M, R, N, false);
      }
    });
  });
  return 0;
}
}  // extern "C"

extern "C" {
// bench.hpp:125-170: the reference's CSV header / row for 17 values
// (7 integers then 10 doubles, in column order); 0 on success
int ref_bench_csv_header(char* out, size_t len) {
  const std::string h = lrbatch::bench_csv_header();
  if (h.size() + 1 > len) return -1;
  std::memcpy(out, h.c_str(), h.size() + 1);
  return 0;
}

int ref_bench_csv_row(const double* v, char* out, size_t len) {
  lrbatch::BenchResult r;
  r.batch_size = size_t(v[0]);
  r.block_size = size_t(v[1]);
  r.rank = size_t(v[2]);
  r.workers = size_t(v[3]);
  r.repetitions = size_t(v[4]);
  r.warmup_reps = size_t(v[5]);
  r.seed = uint64_t(v[6]);
  r.wall_seconds = v[7];
  r.gflops_rate = v[8];
  r.bandwidth_overlapped = v[9];
  r.bandwidth_nonoverlapped = v[10];
  r.pack_small_seconds = v[11];
  r.pack_skinny_seconds = v[12];
  r.kernel_seconds = v[13];
  r.other_seconds = v[14];
  r.baseline_seconds = v[15];
  r.speedup = v[16];
  const std::string row = lrbatch::bench_csv_row(r);
  if (row.size() + 1 > len) return -1;
  std::memcpy(out, row.c_str(), row.size() + 1);
  return 0;
}

// gflops / bandwidth_overlapped_gib_s / bandwidth_nonoverlapped_gib_s and
// median_of (bench.hpp:21-88)
int ref_bench_rates(uint64_t batch, uint64_t rank, uint64_t block, double seconds, double* out) {
  try {
    out[0] = lrbatch::gflops(batch, rank, block, seconds);
    out[1] = lrbatch::bandwidth_overlapped_gib_s(batch, rank, block, seconds);
    out[2] = lrbatch::bandwidth_nonoverlapped_gib_s(batch, rank, block, seconds);
  } catch (...) {
    return -1;
  }
  return 0;
}

double ref_median_of(const double* v, int64_t n) {
  return lrbatch::median_of(std::vector<double>(v, v + n));
}
}  // extern "C"
