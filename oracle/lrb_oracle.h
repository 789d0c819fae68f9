/*
 * lrb_oracle.h — CPU oracle for the batched FP64 GEMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. The product path (liblrb.so) has no CPU
 * fallback and never links or calls this code.
 *
 * Parity is PINNED: the restatement is checked bitwise against the
 * reference's own gemm_naive_raw compiled from /root/reference
 * (oracle/_ref/liblrb_ref.so, recipe in the top-level Makefile) and against
 * the golden vectors in tests/golden/ generated from that build.
 */
#ifndef LRB_ORACLE_H
#define LRB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rounding modes of the batched oracle */
#define ORACLE_FMA_CHAIN 0    /* one fma() per k step: what the B200 kernels compute */
#define ORACLE_REF_COMPILED 1 /* the reference binary's rounding (see oracle_gemm_naive_raw) */

/* Restates lrbatch::gemm_naive_raw (reference proj/include/lrbatch/dense.hpp:43-56):
 * row-major c(m x n) = [c] + a(m x k) * b(k x n); i -> j -> p loops, p ascending,
 * sum starts at 0 or c[i*n+j]; flops += 2 per multiply-add when non-null.
 * Rounding follows the reference as GCC 13 -O3 compiles it: products rounded
 * separately and added in p order, except a fused last step when k is odd
 * (flops == NULL); fully unfused when flops != NULL. Bitwise equal to
 * oracle/_ref (tests/test_oracle.py). */
void oracle_gemm_naive_raw(const double* a, const double* b, double* c, size_t m, size_t k,
                           size_t n, int accumulate, uint64_t* flops);

/* The same arithmetic per item of a strided batch, in either storage order and
 * with transposes, i.e. the semantics of lrb_dgemm_strided_batched. Each C
 * entry is accumulated over ascending p from 0 or C, rounded per `mode`.
 * Items are split contiguously over `threads` workers like the reference's
 * naive_multiply_batch (bench.hpp:55-77). Returns 0, or -1 on bad arguments. */
int oracle_dgemm_strided(int mode, char order, char opA, char opB, int64_t m, int64_t n, int64_t k,
                         double beta, const double* A, int64_t lda, int64_t strideA,
                         const double* B, int64_t ldb, int64_t strideB, double* C, int64_t ldc,
                         int64_t strideC, int64_t batch, int threads);

/* pointer-array form (per-item dims and leading dimensions) */
int oracle_dgemm_ptr(int mode, char order, char opA, char opB, int64_t batch, const int64_t* m,
                     const int64_t* n, const int64_t* k, const double* const* A,
                     const int64_t* lda, const double* const* B, const int64_t* ldb,
                     double* const* C, const int64_t* ldc, double beta, int threads);

/* host twin of lrb_fill_uniform (include/lrb_rng.h generator) */
void oracle_fill_uniform(double* dst, int64_t rows, int64_t cols, int64_t ld, int64_t stride,
                         int64_t batch, uint64_t seed, uint32_t role, int64_t item_offset);

/* Componentwise FP64 bound of BASELINE.json for one item:
 *   |C - C_ref| <= 4 * k * 2^-52 * (|op(A)| |op(B)|)   (+ |C0| term when beta = 1)
 * Computes |op(A)|*|op(B)| with a second naive pass on absolute values.
 * Returns the number of violating entries; *max_ratio = max |C-C_ref| / bound
 * (entries with bound 0 must match exactly; a mismatch there counts as a
 * violation and sets *max_ratio to +inf). C0 may be NULL when beta = 0. */
int64_t oracle_check_bound(char order, char opA, char opB, int64_t m, int64_t n, int64_t k,
                           double beta, const double* A, int64_t lda, const double* B, int64_t ldb,
                           const double* C0, const double* C, const double* Cref, int64_t ldc,
                           double* max_ratio);

/* The paper's batched low-rank product G = A_X (A_Vt B_U) B_X over a
 * LowRankBatch (row-major roles packed contiguously; rank_a == rank_b), as the
 * reference's oracle computes it: three naive products with materialised
 * intermediates (low_rank.hpp:73-87), items split over `threads` like
 * naive_multiply_batch (bench.hpp:55-77). Rounded per `mode`. */
int oracle_lowrank_batch(int mode, int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                         const double* b_u, const double* a_x, const double* b_x, double* g,
                         int threads);

/* BLR multi-RHS matvec, restating blr_matvec_naive (blr.hpp:179-202). */
int oracle_blr_matvec(int mode, int64_t n, int64_t block, int64_t rank, const double* diag,
                      const double* u, const double* x, const double* vt, const double* rhs,
                      int64_t nrhs, double* y);
int oracle_lowrank_expand(int mode, int64_t batch, int64_t m, int64_t n, int64_t r,
                          const double* u, int64_t su, const double* x, int64_t sx,
                          const double* vt, int64_t svt, double* out, int64_t ldo, int64_t so);
int oracle_blr_reconstruct(int mode, int64_t n, int64_t block, int64_t rank, const double* diag,
                           const double* u, const double* x, const double* vt, double* out);

#ifdef __cplusplus
}
#endif

#endif /* LRB_ORACLE_H */
