/*
 * lrb_oracle.c — CPU restatement of the reference's hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY (see lrb_oracle.h): the checker for liblrb.so,
 * loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
 *
 * Compiled with -ffp-contract=off so every rounding is spelled out in the
 * source: explicit fma() where the reference binary fuses, separate multiply
 * and add where it does not (see ref_dot).
 */
#include "lrb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "lrb_rng.h"

/* One reference dot product, rounded the way the reference binary rounds it.
 * Source (dense.hpp:46-50):  sum = acc ? c : 0;  for p < k: sum += a[p] * b[p].
 * GCC 13.3 at -O3 (-march=native or x86-64-v3; proj/CMakeLists.txt:13-20)
 * versions that loop on `flops`:
 *   flops == NULL: the p loop is vectorised two-wide with an in-order
 *     reduction: vmulpd forms two separately rounded products, two vaddsd add
 *     them to sum in p order; an odd last p goes through the scalar epilogue,
 *     which is contracted to vfmadd231sd.
 *   flops != NULL: scalar vmulsd + vaddsd for every p (no contraction).
 * (disassembly probe: `objdump -d oracle/_ref/liblrb_ref.so`.) */
static inline double ref_dot(const double* a, int64_t sa, const double* b, int64_t sb, int64_t k,
                             double sum, int unfused_all) {
  int64_t p = 0;
  const int64_t kv = unfused_all ? k : (k & ~(int64_t)1);
  for (; p < kv; ++p) {
    const double prod = a[p * sa] * b[p * sb];
    sum = sum + prod;
  }
  for (; p < k; ++p) sum = fma(a[p * sa], b[p * sb], sum);
  return sum;
}

/* reference proj/include/lrbatch/dense.hpp:43-56, as compiled (see ref_dot) */
void oracle_gemm_naive_raw(const double* a, const double* b, double* c, size_t m, size_t k,
                           size_t n, int accumulate, uint64_t* flops) {
  for (size_t i = 0; i < m; ++i) {
    for (size_t j = 0; j < n; ++j) {
      double sum = accumulate ? c[i * n + j] : 0.0;
      sum = ref_dot(a + i * k, 1, b + j, (int64_t)n, (int64_t)k, sum, flops != NULL);
      if (flops) *flops += 2 * (uint64_t)k;
      c[i * n + j] = sum;
    }
  }
}

static int is_row(char o) { return o == 'R' || o == 'r'; }
static int is_t(char o) { return o == 'T' || o == 't'; }
static int ok_order(char o) { return o == 'C' || o == 'c' || o == 'R' || o == 'r'; }
static int ok_op(char o) { return o == 'N' || o == 'n' || o == 'T' || o == 't'; }

/* stored element (r, c) of a matrix in `order` with leading dimension ld */
static inline double at(const double* X, int row, int64_t r, int64_t c, int64_t ld) {
  return row ? X[r * ld + c] : X[r + c * ld];
}

/* one item: C = op(A) op(B) + beta C over ascending p.
 * mode ORACLE_FMA_CHAIN: one fma() per p (the device kernels' rounding);
 * mode ORACLE_REF_COMPILED: ref_dot's rounding (the reference binary). */
static void item_gemm(int mode, int row, int ta, int tb, int64_t m, int64_t n, int64_t k,
                      int beta_one, const double* A, int64_t lda, const double* B, int64_t ldb,
                      double* C, int64_t ldc) {
  /* Strided operand rows are first gathered into contiguous scratch (exact
   * copies, same values, same summation order) so the p loop is unit-stride. */
  const int64_t sa0 = ta ? (row ? lda : 1) : (row ? 1 : lda);
  const int64_t sb0 = tb ? (row ? 1 : ldb) : (row ? ldb : 1);
  double* at_s = NULL; /* op(A) as m x k row-major */
  double* bt_s = NULL; /* op(B)^T as n x k row-major */
  if (sa0 != 1 && m > 0 && k > 0) {
    at_s = (double*)malloc(sizeof(double) * (size_t)(m * k));
    for (int64_t i = 0; i < m; ++i) {
      const double* a_i = ta ? (row ? A + i : A + i * lda) : (row ? A + i * lda : A + i);
      for (int64_t p = 0; p < k; ++p) at_s[i * k + p] = a_i[p * sa0];
    }
  }
  if (sb0 != 1 && n > 0 && k > 0) {
    bt_s = (double*)malloc(sizeof(double) * (size_t)(n * k));
    for (int64_t j = 0; j < n; ++j) {
      const double* b_j = tb ? (row ? B + j * ldb : B + j) : (row ? B + j : B + j * ldb);
      for (int64_t p = 0; p < k; ++p) bt_s[j * k + p] = b_j[p * sb0];
    }
  }
  for (int64_t i = 0; i < m; ++i) {
    /* op(A)(i, p) = a_i[p * sa] */
    const double* a_i =
        at_s ? at_s + i * k : (ta ? (row ? A + i : A + i * lda) : (row ? A + i * lda : A + i));
    const int64_t sa = at_s ? 1 : sa0;
    for (int64_t j = 0; j < n; ++j) {
      /* op(B)(p, j) = b_j[p * sb] */
      const double* b_j =
          bt_s ? bt_s + j * k : (tb ? (row ? B + j * ldb : B + j) : (row ? B + j : B + j * ldb));
      const int64_t sb = bt_s ? 1 : sb0;
      double* cij = row ? &C[i * ldc + j] : &C[i + j * ldc];
      double sum = beta_one ? *cij : 0.0;
      if (mode == ORACLE_REF_COMPILED) {
        sum = ref_dot(a_i, sa, b_j, sb, k, sum, 0);
      } else {
        for (int64_t p = 0; p < k; ++p) sum = fma(a_i[p * sa], b_j[p * sb], sum);
      }
      *cij = sum;
    }
  }
  free(at_s);
  free(bt_s);
}

typedef struct {
  int kind; /* 0 strided, 1 ptr */
  int mode;
  int row, ta, tb, beta_one;
  int64_t m, n, k;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  const int64_t *pm, *pn, *pk, *plda, *pldb, *pldc;
  const double* const* pA;
  const double* const* pB;
  double* const* pC;
  int64_t begin, end;
} job_t;

static void run_items(const job_t* j) {
  for (int64_t it = j->begin; it < j->end; ++it) {
    if (j->kind == 0)
      item_gemm(j->mode, j->row, j->ta, j->tb, j->m, j->n, j->k, j->beta_one, j->A + it * j->sA, j->lda,
                j->B + it * j->sB, j->ldb, j->C + it * j->sC, j->ldc);
    else
      item_gemm(j->mode, j->row, j->ta, j->tb, j->pm[it], j->pn[it], j->pk[it], j->beta_one, j->pA[it],
                j->plda[it], j->pB[it], j->pldb[it], j->pC[it], j->pldc[it]);
  }
}

static void* worker(void* arg) {
  run_items((const job_t*)arg);
  return NULL;
}

/* contiguous split over workers exactly like naive_multiply_batch (bench.hpp:59-76) */
static void fan_out(const job_t* proto, int64_t batch, int threads) {
  if (threads < 1) threads = 1;
  if (threads > batch) threads = (int)(batch > 0 ? batch : 1);
  if (threads == 1) {
    job_t j = *proto;
    j.begin = 0;
    j.end = batch;
    run_items(&j);
    return;
  }
  const int64_t per = (batch + threads - 1) / threads;
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int w = 0; w < threads; ++w) {
    jobs[w] = *proto;
    int64_t b = (int64_t)w * per;
    if (b > batch) b = batch;
    int64_t e = b + per;
    if (e > batch) e = batch;
    jobs[w].begin = b;
    jobs[w].end = e;
  }
  for (int w = 1; w < threads; ++w) pthread_create(&tids[w], NULL, worker, &jobs[w]);
  run_items(&jobs[0]);
  for (int w = 1; w < threads; ++w) pthread_join(tids[w], NULL);
  free(jobs);
  free(tids);
}

int oracle_dgemm_strided(int mode, char order, char opA, char opB, int64_t m, int64_t n, int64_t k,
                         double beta, const double* A, int64_t lda, int64_t strideA,
                         const double* B, int64_t ldb, int64_t strideB, double* C, int64_t ldc,
                         int64_t strideC, int64_t batch, int threads) {
  if (!ok_order(order) || !ok_op(opA) || !ok_op(opB)) return -1;
  if (mode != ORACLE_FMA_CHAIN && mode != ORACLE_REF_COMPILED) return -1;
  if (m < 0 || n < 0 || k < 0 || batch < 0 || !(beta == 0.0 || beta == 1.0)) return -1;
  job_t j;
  memset(&j, 0, sizeof j);
  j.kind = 0;
  j.mode = mode;
  j.row = is_row(order);
  j.ta = is_t(opA);
  j.tb = is_t(opB);
  j.beta_one = beta == 1.0;
  j.m = m;
  j.n = n;
  j.k = k;
  j.A = A;
  j.lda = lda;
  j.sA = strideA;
  j.B = B;
  j.ldb = ldb;
  j.sB = strideB;
  j.C = C;
  j.ldc = ldc;
  j.sC = strideC;
  fan_out(&j, batch, threads);
  return 0;
}

int oracle_dgemm_ptr(int mode, char order, char opA, char opB, int64_t batch, const int64_t* m,
                     const int64_t* n, const int64_t* k, const double* const* A,
                     const int64_t* lda, const double* const* B, const int64_t* ldb,
                     double* const* C, const int64_t* ldc, double beta, int threads) {
  if (!ok_order(order) || !ok_op(opA) || !ok_op(opB) || batch < 0) return -1;
  if (mode != ORACLE_FMA_CHAIN && mode != ORACLE_REF_COMPILED) return -1;
  if (!(beta == 0.0 || beta == 1.0)) return -1;
  job_t j;
  memset(&j, 0, sizeof j);
  j.kind = 1;
  j.mode = mode;
  j.row = is_row(order);
  j.ta = is_t(opA);
  j.tb = is_t(opB);
  j.beta_one = beta == 1.0;
  j.pm = m;
  j.pn = n;
  j.pk = k;
  j.pA = A;
  j.plda = lda;
  j.pB = B;
  j.pldb = ldb;
  j.pC = C;
  j.pldc = ldc;
  fan_out(&j, batch, threads);
  return 0;
}

void oracle_fill_uniform(double* dst, int64_t rows, int64_t cols, int64_t ld, int64_t stride,
                         int64_t batch, uint64_t seed, uint32_t role, int64_t item_offset) {
  const uint64_t key = lrb_stream_key(seed, role);
  for (int64_t it = 0; it < batch; ++it)
    for (int64_t c = 0; c < cols; ++c)
      for (int64_t r = 0; r < rows; ++r)
        dst[it * stride + c * ld + r] =
            lrb_uniform(key, (uint64_t)(item_offset + it), (uint64_t)(r + c * rows));
}

int64_t oracle_check_bound(char order, char opA, char opB, int64_t m, int64_t n, int64_t k,
                           double beta, const double* A, int64_t lda, const double* B, int64_t ldb,
                           const double* C0, const double* C, const double* Cref, int64_t ldc,
                           double* max_ratio) {
  const int row = is_row(order), ta = is_t(opA), tb = is_t(opB);
  const double u = ldexp(1.0, -52);
  int64_t bad = 0;
  double worst = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double mag = 0.0;
      for (int64_t p = 0; p < k; ++p) {
        const double a = ta ? at(A, row, p, i, lda) : at(A, row, i, p, lda);
        const double b = tb ? at(B, row, j, p, ldb) : at(B, row, p, j, ldb);
        mag += fabs(a) * fabs(b);
      }
      const int64_t off = row ? i * ldc + j : i + j * ldc;
      double bound = 4.0 * (double)k * u * mag;
      if (beta == 1.0 && C0) bound = 4.0 * (double)(k + 1) * u * (mag + fabs(C0[off]));
      const double err = fabs(C[off] - Cref[off]);
      if (C[off] != C[off] || Cref[off] != Cref[off]) { /* NaN */
        ++bad;
        worst = INFINITY;
        continue;
      }
      if (bound == 0.0) {
        if (err != 0.0) {
          ++bad;
          worst = INFINITY;
        }
        continue;
      }
      const double ratio = err / bound;
      if (ratio > worst) worst = ratio;
      if (ratio > 1.0) ++bad;
    }
  }
  if (max_ratio) *max_ratio = worst;
  return bad;
}

/* ------------------------------------------------------------------------
 * The paper's batched low-rank product (reference low_rank.hpp:73-87,
 * reference_item :179-184, naive_multiply_batch bench.hpp:55-77):
 *   C = A_Vt (r x b) B_U (b x r); E = A_X C; G = E B_X — three naive
 *   row-major products with materialised intermediates, per item of a
 *   LowRankBatch (roles packed contiguously, item i at base + i*rows*cols). */
typedef struct {
  int mode;
  int64_t block, rank;
  const double *a_vt, *b_u, *a_x, *b_x;
  double* g;
  int64_t begin, end;
} lr_job_t;

static void lr_gemm(int mode, const double* a, const double* b, double* c, int64_t m, int64_t k,
                    int64_t n) {
  /* gemm_naive_raw(a, b, c, m, k, n, false) (dense.hpp:43-56) in `mode` rounding */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double sum = 0.0;
      if (mode == ORACLE_REF_COMPILED)
        sum = ref_dot(a + i * k, 1, b + j, n, k, sum, 0);
      else
        for (int64_t p = 0; p < k; ++p) sum = fma(a[i * k + p], b[p * n + j], sum);
      c[i * n + j] = sum;
    }
}

static void* lr_worker(void* arg) {
  const lr_job_t* j = (const lr_job_t*)arg;
  const int64_t r = j->rank, b = j->block;
  double* cs = (double*)malloc(sizeof(double) * (size_t)(r * r));
  double* es = (double*)malloc(sizeof(double) * (size_t)(r * r));
  for (int64_t it = j->begin; it < j->end; ++it) {
    lr_gemm(j->mode, j->a_vt + it * r * b, j->b_u + it * b * r, cs, r, b, r);
    lr_gemm(j->mode, j->a_x + it * r * r, cs, es, r, r, r);
    lr_gemm(j->mode, es, j->b_x + it * r * r, j->g + it * r * r, r, r, r);
  }
  free(cs);
  free(es);
  return NULL;
}

int oracle_lowrank_batch(int mode, int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                         const double* b_u, const double* a_x, const double* b_x, double* g,
                         int threads) {
  if (batch < 0 || block < 1 || rank < 1) return -1;
  if (mode != ORACLE_FMA_CHAIN && mode != ORACLE_REF_COMPILED) return -1;
  if (threads < 1) threads = 1;
  if (threads > batch) threads = (int)(batch > 0 ? batch : 1);
  const int64_t per = (batch + threads - 1) / threads; /* bench.hpp:69-75 split */
  lr_job_t* jobs = (lr_job_t*)malloc(sizeof(lr_job_t) * (size_t)threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int w = 0; w < threads; ++w) {
    int64_t bg = (int64_t)w * per;
    if (bg > batch) bg = batch;
    int64_t en = bg + per;
    if (en > batch) en = batch;
    lr_job_t jb = {mode, block, rank, a_vt, b_u, a_x, b_x, g, bg, en};
    jobs[w] = jb;
  }
  for (int w = 1; w < threads; ++w) pthread_create(&tids[w], NULL, lr_worker, &jobs[w]);
  lr_worker(&jobs[0]);
  for (int w = 1; w < threads; ++w) pthread_join(tids[w], NULL);
  free(jobs);
  free(tids);
  return 0;
}

/* ------------------------------------------------------------------------
 * BLR multi-RHS matvec, restating blr_matvec_naive (reference
 * blr.hpp:179-202): y_i = D_i rhs_i for every tile, then for i, j != i
 * ascending: vt_x = Vt_ij rhs_j; x_vt_x = X_ij vt_x; y_i += U_ij x_vt_x.
 * Inputs in the reference layout (BlrMatrix: diagonal tiles, off-diagonal
 * LowRankOperands row-major over (i, j != i)); rhs and y row-major n x nrhs. */
static void gemm_acc(int mode, const double* a, const double* b, double* c, int64_t m, int64_t k,
                     int64_t n, int acc) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double sum = acc ? c[i * n + j] : 0.0;
      if (mode == ORACLE_REF_COMPILED)
        sum = ref_dot(a + i * k, 1, b + j, n, k, sum, 0);
      else
        for (int64_t p = 0; p < k; ++p) sum = fma(a[i * k + p], b[p * n + j], sum);
      c[i * n + j] = sum;
    }
}

int oracle_blr_matvec(int mode, int64_t n, int64_t block, int64_t rank, const double* diag,
                      const double* u, const double* x, const double* vt, const double* rhs,
                      int64_t nrhs, double* y) {
  if (block < 1 || n % block || rank < 1 || nrhs < 1) return -1;
  const int64_t T = n / block, b = block, r = rank;
  memset(y, 0, sizeof(double) * (size_t)(n * nrhs));
  for (int64_t i = 0; i < T; ++i)
    gemm_acc(mode, diag + i * b * b, rhs + i * b * nrhs, y + i * b * nrhs, b, b, nrhs, 1);
  double* vt_x = (double*)malloc(sizeof(double) * (size_t)(r * nrhs));
  double* x_vt_x = (double*)malloc(sizeof(double) * (size_t)(r * nrhs));
  for (int64_t i = 0; i < T; ++i)
    for (int64_t j = 0; j < T; ++j) {
      if (i == j) continue;
      const int64_t o = i * (T - 1) + (j < i ? j : j - 1);
      gemm_acc(mode, vt + o * r * b, rhs + j * b * nrhs, vt_x, r, b, nrhs, 0);
      gemm_acc(mode, x + o * r * r, vt_x, x_vt_x, r, r, nrhs, 0);
      gemm_acc(mode, u + o * b * r, x_vt_x, y + i * b * nrhs, b, r, nrhs, 1);
    }
  free(vt_x);
  free(x_vt_x);
  return 0;
}

/* ------------------------------------------------------------------------
 * Low-rank expansion out_i = (U_i X_i) Vt_i of a batch of LowRankOperands
 * (low_rank.hpp:16-63), restating the per-tile expansion inside
 * BlrMatrix::reconstruct_dense (blr.hpp:75-78): UX = dense_gemm_naive(U, X),
 * then tile = dense_gemm_naive(UX, Vt), each gemm_naive_raw without a flop
 * counter (dense.hpp:58-77). Items row-major at base + it*stride; out_i has
 * leading dimension ldo. */
int oracle_lowrank_expand(int mode, int64_t batch, int64_t m, int64_t n, int64_t r,
                          const double* u, int64_t su, const double* x, int64_t sx,
                          const double* vt, int64_t svt, double* out, int64_t ldo, int64_t so) {
  if (batch < 0 || m < 0 || n < 0 || r < 1 || ldo < n) return -1;
  double* ux = (double*)malloc(sizeof(double) * (size_t)(m * r + 1));
  double* tile = (double*)malloc(sizeof(double) * (size_t)(m * n + 1));
  for (int64_t it = 0; it < batch; ++it) {
    gemm_acc(mode, u + it * su, x + it * sx, ux, m, r, r, 0);
    gemm_acc(mode, ux, vt + it * svt, tile, m, r, n, 0);
    for (int64_t row = 0; row < m; ++row)
      memcpy(out + it * so + row * ldo, tile + row * n, sizeof(double) * (size_t)n);
  }
  free(ux);
  free(tile);
  return 0;
}

/* BlrMatrix::reconstruct_dense (blr.hpp:62-86): the n x n row-major matrix,
 * diagonal tiles copied, off-diagonal tiles (U X) Vt. */
int oracle_blr_reconstruct(int mode, int64_t n, int64_t block, int64_t rank, const double* diag,
                           const double* u, const double* x, const double* vt, double* out) {
  if (block < 1 || n % block || rank < 1) return -1;
  const int64_t T = n / block, b = block, r = rank;
  for (int64_t ti = 0; ti < T; ++ti)
    for (int64_t tj = 0; tj < T; ++tj) {
      double* dst = out + ti * b * n + tj * b;
      if (ti == tj) {
        for (int64_t row = 0; row < b; ++row)
          memcpy(dst + row * n, diag + ti * b * b + row * b, sizeof(double) * (size_t)b);
      } else {
        const int64_t o = ti * (T - 1) + (tj < ti ? tj : tj - 1);
        oracle_lowrank_expand(mode, 1, b, b, r, u + o * b * r, 0, x + o * r * r, 0,
                              vt + o * r * b, 0, dst, n, 0);
      }
    }
  return 0;
}
