/*
 * lrb.h — C-ABI of the B200-native batched FP64 GEMM hot path (liblrb.so).
 *
 * The reference (lrbatch, header-only C++20) computes every BASELINE shape with
 * its oracle primitive
 *     void lrbatch::gemm_naive_raw(const double* a, const double* b, double* c,
 *                                  size_t m, size_t k, size_t n, bool accumulate,
 *                                  uint64_t* flops = nullptr);
 * (reference: proj/include/lrbatch/dense.hpp:43-56), called item by item over
 * batches packed with the LowRankBatch convention "item i of a role starts at
 * base + i*rows*cols, row-major per item" (low_rank.hpp:147-158), e.g. at the
 * BLR diagonal step (blr.hpp:149-153) and the tile expansion (blr.hpp:75-78).
 * This header is the drop-in boundary for that path: plain pointers and sizes,
 * status codes instead of exceptions, no CUDA or torch types.
 *
 * Conventions
 *  - Results equal the reference FMA chain: every C entry is accumulated in
 *    ascending k from 0 (beta = 0) or from the old C (beta = 1), one fused
 *    multiply-add per k. The kernels use FP64 DMMA/DFMA, which round exactly
 *    like that chain, so results are bitwise equal to gemm_naive_raw compiled
 *    with FMA contraction (what the reference's -O3 -march=native build does).
 *  - order 'C' = column-major (BASELINE), 'R' = row-major (the reference).
 *  - beta must be 0 or 1: it is the reference's `accumulate` flag. With beta
 *    = 0, C is never read.
 *  - Device-pointer calls are asynchronous on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream). Host-buffer calls (`_host`,
 *    lrb_gemm_naive_raw) are synchronous like the reference.
 *  - Errors: every call returns lrb_status; lrb_last_error(ctx) holds the
 *    message. LRB_ERR_SHAPE mirrors the reference ShapeError (common.hpp:19-22)
 *    and names the offending pair the way dense_gemm_naive does
 *    (dense.hpp:58-69), LRB_ERR_CAPACITY mirrors CapacityError (common.hpp:24-27).
 *  - There is no CPU fallback: without a usable sm_100 device, lrb_create
 *    fails with LRB_ERR_NO_DEVICE.
 */
#ifndef LRB_H
#define LRB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* the library is built with -fvisibility=hidden; these are its only exports */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LRB_VERSION_STRING "lrb-b200 0.1.0"

typedef enum lrb_status {
  LRB_OK = 0,
  LRB_ERR_SHAPE = 1,       /* dimension / leading-dimension / stride invariant violated */
  LRB_ERR_CAPACITY = 2,    /* workspace or device memory exhausted */
  LRB_ERR_ARG = 3,         /* bad enum value, null pointer, bad handle */
  LRB_ERR_CUDA = 4,        /* CUDA runtime error (message carries cudaGetErrorString) */
  LRB_ERR_UNSUPPORTED = 5, /* valid request outside what this build implements */
  LRB_ERR_NO_DEVICE = 6,   /* no CUDA device / not sm_100 */
  LRB_ERR_IO = 7,          /* file cannot be opened / written (reference IoError) */
  LRB_ERR_PARSE = 8        /* malformed batch file (reference ParseError) */
} lrb_status;

typedef struct lrb_ctx lrb_ctx;           /* one per (host thread, device) */
typedef struct lrb_ptr_plan lrb_ptr_plan; /* descriptor of a pointer-array batch */

/* ---------------------------------------------------------------- context */
lrb_status lrb_create(int device, lrb_ctx** out);
lrb_status lrb_destroy(lrb_ctx* ctx);
const char* lrb_last_error(const lrb_ctx* ctx); /* ctx may be NULL: thread-local last error */
const char* lrb_version(void);
int lrb_device_count(void); /* 0 when no driver / no device; never fails */
/* the device's name (cudaGetDeviceProperties), NUL-terminated into buf */
lrb_status lrb_device_name(int device, char* buf, size_t len);
int lrb_ctx_device(const lrb_ctx* ctx);
int lrb_ctx_sm_count(const lrb_ctx* ctx);
/* number of kernels this context has launched so far (GEMM + fill + flush) */
uint64_t lrb_launch_count(const lrb_ctx* ctx);
/* the kernel (variant id, lrb_variant_name) that served this context's last
   strided GEMM, -1 before the first one */
int lrb_last_variant(const lrb_ctx* ctx);

/* ------------------------------------------------ memory / stream helpers */
lrb_status lrb_malloc(lrb_ctx* ctx, size_t bytes, void** dptr);
lrb_status lrb_free(lrb_ctx* ctx, void* dptr);
lrb_status lrb_host_alloc(lrb_ctx* ctx, size_t bytes, void** hptr); /* pinned */
lrb_status lrb_host_free(lrb_ctx* ctx, void* hptr);
lrb_status lrb_memcpy_h2d(lrb_ctx* ctx, void* dst, const void* src, size_t bytes);
lrb_status lrb_memcpy_d2h(lrb_ctx* ctx, void* dst, const void* src, size_t bytes);
lrb_status lrb_memset(lrb_ctx* ctx, void* dptr, int value, size_t bytes);
lrb_status lrb_stream_create(lrb_ctx* ctx, void** stream);
lrb_status lrb_stream_destroy(lrb_ctx* ctx, void* stream);
lrb_status lrb_stream_sync(lrb_ctx* ctx, void* stream);
lrb_status lrb_device_sync(lrb_ctx* ctx);
/* free / total device memory in bytes */
lrb_status lrb_mem_info(lrb_ctx* ctx, size_t* free_bytes, size_t* total_bytes);

/* CUDA events for device-side timing on the launching stream */
lrb_status lrb_event_create(lrb_ctx* ctx, void** ev);
lrb_status lrb_event_destroy(lrb_ctx* ctx, void* ev);
lrb_status lrb_event_record(lrb_ctx* ctx, void* ev, void* stream);
lrb_status lrb_event_elapsed_ms(lrb_ctx* ctx, void* ev_start, void* ev_end, float* ms);
/* write a buffer larger than L2 on `stream` (timing hygiene between reps) */
lrb_status lrb_l2_flush(lrb_ctx* ctx, void* stream);
/* read a clean buffer of twice the L2 size on `stream`: the next kernel
   starts with none of its data in L2 and no dirty lines to write back
   (a cold call without lrb_l2_flush's write-back tail) */
lrb_status lrb_l2_evict(lrb_ctx* ctx, void* stream);

/* ------------------------------------------------------------- hot path */
/*
 * Strided batch: item i uses A + i*strideA, B + i*strideB, C + i*strideC
 * (elements). C_i = op(A_i) * op(B_i) + beta * C_i with op(A) m x k,
 * op(B) k x n, C m x n, all in `order`. The reference's LowRankBatch packing
 * is strideX = rows*cols, ldX = cols (order 'R'); BASELINE's is
 * strideX = rows*cols, ldX = rows (order 'C').
 * Replaces: lrbatch::gemm_naive_raw called per item (dense.hpp:43-56), e.g. the
 * BLR diagonal loop (blr.hpp:149-153) and naive_multiply_batch's per-item
 * fan-out (bench.hpp:55-77).
 */
lrb_status lrb_dgemm_strided_batched(lrb_ctx* ctx, char order, char opA, char opB,
                                     int64_t m, int64_t n, int64_t k, double beta,
                                     const double* A, int64_t lda, int64_t strideA,
                                     const double* B, int64_t ldb, int64_t strideB,
                                     double* C, int64_t ldc, int64_t strideC,
                                     int64_t batch, void* stream);

/*
 * Pointer-array / variable-size batch. Dimension and leading-dimension arrays
 * are HOST arrays of length `batch`; A/B/C are HOST arrays of DEVICE pointers.
 * The plan buckets items by kernel variant, builds per-variant tile lists
 * (largest k first) and uploads them once; execute is then one launch per
 * non-empty variant. Replaces: per-item gemm_naive_raw over independently
 * allocated blocks (blr.hpp:141-175's diagonal and scatter steps).
 */
lrb_status lrb_ptr_plan_create(lrb_ctx* ctx, char order, char opA, char opB, int64_t batch,
                               const int64_t* m, const int64_t* n, const int64_t* k,
                               const double* const* A, const int64_t* lda,
                               const double* const* B, const int64_t* ldb,
                               double* const* C, const int64_t* ldc, double beta,
                               lrb_ptr_plan** out);
lrb_status lrb_ptr_plan_execute(lrb_ctx* ctx, const lrb_ptr_plan* plan, void* stream);
lrb_status lrb_ptr_plan_destroy(lrb_ctx* ctx, lrb_ptr_plan* plan);
/* number of kernel launches one execute performs */
int lrb_ptr_plan_launches(const lrb_ptr_plan* plan);
/* one-shot create + execute + (stream-synchronised) destroy */
lrb_status lrb_dgemm_ptr_batched(lrb_ctx* ctx, char order, char opA, char opB, int64_t batch,
                                 const int64_t* m, const int64_t* n, const int64_t* k,
                                 const double* const* A, const int64_t* lda,
                                 const double* const* B, const int64_t* ldb,
                                 double* const* C, const int64_t* ldc, double beta,
                                 void* stream);

/*
 * Pointer-array batch whose descriptor arrays (m, n, k, A, lda, B, ldb, C,
 * ldc, each of length `batch`) live in DEVICE memory, e.g. built by the
 * caller's own kernels (SURVEY §8(b)'s lrb_dgemm_ptr_batched). No host round
 * trip: descriptor checks, tensor-map construction (tensormap.replace), cost
 * ordering and tile prefix sums run as small kernels on `stream`, followed by
 * the single-launch variable-size kernel and a generic kernel for items TMA
 * cannot address. Asynchronous and capturable in lrb_graph_*. Items with
 * invalid descriptors (negative extents, too-small leading dimensions, null
 * operands, more than 65535 x 64 rows or columns) are skipped; when `info`
 * (a DEVICE int64_t[2]) is non-null it receives {number of skipped items,
 * first skipped index or -1}. Replaces: per-item gemm_naive_raw over blocks a
 * GPU-resident BLR caller enumerates (blr.hpp:141-175).
 */
lrb_status lrb_dgemm_ptr_batched_device(lrb_ctx* ctx, char order, char opA, char opB,
                                        int64_t batch, const int64_t* m, const int64_t* n,
                                        const int64_t* k, const double* const* A,
                                        const int64_t* lda, const double* const* B,
                                        const int64_t* ldb, double* const* C,
                                        const int64_t* ldc, double beta, int64_t* info,
                                        void* stream);

/* ------------------------------------------------ host-buffer entry points */
/*
 * Drop-in for lrbatch::gemm_naive_raw (dense.hpp:43-45): row-major HOST
 * buffers a (m x k), b (k x n), c (m x n); accumulate = reference flag;
 * `flops` (nullable) is incremented by 2*m*n*k exactly like the reference's
 * in-loop counter. Synchronous.
 */
lrb_status lrb_gemm_naive_raw(lrb_ctx* ctx, const double* a, const double* b, double* c,
                              size_t m, size_t k, size_t n, int accumulate, uint64_t* flops);
/*
 * Same contract as lrb_dgemm_strided_batched but on HOST buffers: the batch
 * is cut into chunks whose H2D copy, kernel and D2H copy are pipelined over
 * three streams. Pinned host memory (lrb_host_alloc) gets full PCIe rate.
 * Synchronous.
 */
lrb_status lrb_dgemm_strided_batched_host(lrb_ctx* ctx, char order, char opA, char opB,
                                          int64_t m, int64_t n, int64_t k, double beta,
                                          const double* A, int64_t lda, int64_t strideA,
                                          const double* B, int64_t ldb, int64_t strideB,
                                          double* C, int64_t ldc, int64_t strideC,
                                          int64_t batch);
/*
 * Pointer-array batch on HOST buffers (the reference's own mode: per-tile
 * gemm_naive_raw calls over separately allocated blocks, blr.hpp:141-175;
 * the per-item fan-out of naive_multiply_batch, bench.hpp:55-77). Same
 * descriptor arrays as lrb_dgemm_ptr_batched, but A[i], B[i], C[i] are host
 * pointers. Items are cut into chunks; within a chunk, operands that lie back
 * to back in host memory move as one copy (input runs may span up to 4 KiB of
 * allocation padding), and each chunk's H2D copy, pointer-array kernels and
 * D2H copy are pipelined over three streams. Pinned memory (lrb_host_alloc)
 * gets full PCIe rate; pageable memory goes through pinned staging.
 * Synchronous.
 */
lrb_status lrb_dgemm_ptr_batched_host(lrb_ctx* ctx, char order, char opA, char opB, int64_t batch,
                                      const int64_t* m, const int64_t* n, const int64_t* k,
                                      const double* const* A, const int64_t* lda,
                                      const double* const* B, const int64_t* ldb,
                                      double* const* C, const int64_t* ldc, double beta);

/* ------------------------------------------- the paper's low-rank product */
/*
 * G_i = A_X_i (A_Vt_i B_U_i) B_X_i over a LowRankBatch (arXiv 2311.07602,
 * Algorithm 1): all matrices row-major, each role packed contiguously with
 * item i at base + i*rows*cols (reference low_rank.hpp:109-176):
 *   a_vt: rank x block, b_u: block x rank, a_x, b_x, g: rank x rank.
 * rank_a == rank_b == rank, as fused_multiply / packed_multiply require
 * (kernels.hpp:133-135, 246-248). G is overwritten (stored once per item).
 * Each product is an in-order FMA chain, i.e. the reference oracle
 * low_rank_multiply_reference_raw (low_rank.hpp:73-87) with fused rounding.
 * One launch for rank <= 32 (a warp per item) and for ranks 64, 96 and 128
 * (a CTA per item, the intermediates on chip); three batched GEMMs otherwise.
 * Replaces: fused_multiply (kernels.hpp:131-161), packed_multiply
 * (kernels.hpp:243-349), naive_multiply_batch (bench.hpp:55-77).
 */
lrb_status lrb_lowrank_multiply(lrb_ctx* ctx, int64_t batch, int64_t block, int64_t rank,
                                const double* a_vt, const double* b_u, const double* a_x,
                                const double* b_x, double* g, void* stream);
/* host-buffer form (synchronous; chunked H2D / kernel / D2H) */
lrb_status lrb_lowrank_multiply_host(lrb_ctx* ctx, int64_t batch, int64_t block, int64_t rank,
                                     const double* a_vt, const double* b_u, const double* a_x,
                                     const double* b_x, double* g);
/* the reference's accounting 4 r^3 + 2 r^2 b (flops_per_item, low_rank.hpp:66-68) */
double lrb_lowrank_flops_per_item(int64_t rank, int64_t block);

/*
 * Low-rank expansion of a batch of LowRankOperands (low_rank.hpp:16-63):
 *   out_i = (U_i X_i) Vt_i        U m x rank, X rank x rank, Vt rank x n,
 * all row-major, item i at base + i*stride; out_i m x n with leading
 * dimension ldo >= n. The reference's per-tile expansion inside
 * BlrMatrix::reconstruct_dense (blr.hpp:75-78: dense_gemm_naive(U, X), then
 * dense_gemm_naive(UX, Vt)) in the same order: UX is formed (rounded) first,
 * each entry an in-order FMA chain. UX lives in the context workspace.
 * Device pointers, asynchronous on `stream`.
 */
lrb_status lrb_lowrank_expand(lrb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t rank,
                              const double* u, int64_t su, const double* x, int64_t sx,
                              const double* vt, int64_t svt, double* out, int64_t ldo,
                              int64_t so, void* stream);

/* ------------------------------------------------- LRBATCH1 batch files */
/*
 * The reference's flat batch file (batch_io.hpp:11-77): "LRBATCH1", uint64
 * batch_size, block_size, rank_a, rank_b, then a_vt, b_u, a_x, b_x as
 * doubles (results not stored). Error texts follow save_batch / load_batch.
 * hdr receives {batch_size, block_size, rank_a, rank_b}. With device_ptrs the
 * role buffers are DEVICE pointers and the payload streams through pinned
 * staging into HBM; otherwise they are host pointers.
 */
lrb_status lrb_batch_file_header(const char* path, int64_t* hdr);
lrb_status lrb_batch_file_load(lrb_ctx* ctx, const char* path, double* a_vt, double* b_u,
                               double* a_x, double* b_x, int device_ptrs);
lrb_status lrb_batch_file_save(lrb_ctx* ctx, const char* path, int64_t batch, int64_t block,
                               int64_t rank_a, int64_t rank_b, const double* a_vt,
                               const double* b_u, const double* a_x, const double* b_x,
                               int device_ptrs);

/* --------------------------------------------- BLR multi-RHS matvec */
/*
 * Weakly admissible block low-rank matrix (reference BlrMatrix,
 * blr.hpp:15-87) held on the device: n = tiles * block; host inputs in the
 * reference's layout — diag: tiles dense block x block tiles; u, x, vt: the
 * tiles*(tiles-1) off-diagonal factors in row-major (i, j != i) order, each
 * row-major (u block x rank, x rank x rank, vt rank x block).
 * lrb_blr_matvec: y = M rhs (blr_matvec, blr.hpp:141-175) for row-major
 * n x nrhs HOST buffers; the _device form takes device buffers and is
 * asynchronous. One persistent launch for up to 16 right-hand sides (block a
 * multiple of 32, rank 4, 8, 16 or 32, 16-byte aligned operands; an odd
 * count, e.g. the plain matvec, runs it on copies padded with one zero
 * column: two small copy kernels around it; 17 to 64 right-hand sides at
 * rank >= 16 run it once per column range of 16), otherwise two
 * batched GEMM launches around one coupling kernel; on the caller's stream,
 * every chain in the reference's order (y_i = D_i rhs_i, then
 * += U_ij X_ij Vt_ij rhs_j for j ascending). The matrix owns a
 * grow-only matvec workspace: eager calls on different streams are ordered
 * through an event, and buffers a captured graph references stay alive
 * until lrb_blr_destroy.
 */
typedef struct lrb_blr lrb_blr;
lrb_status lrb_blr_create(lrb_ctx* ctx, int64_t n, int64_t block, int64_t rank, const double* diag,
                          const double* u, const double* x, const double* vt, lrb_blr** out);
lrb_status lrb_blr_matvec(lrb_ctx* ctx, lrb_blr* m, const double* rhs, int64_t nrhs, double* y);
lrb_status lrb_blr_matvec_device(lrb_ctx* ctx, lrb_blr* m, const double* rhs, int64_t nrhs,
                                 double* y, void* stream);
lrb_status lrb_blr_destroy(lrb_ctx* ctx, lrb_blr* m);
/*
 * Exact dense assembly of the whole n x n matrix, row-major
 * (BlrMatrix::reconstruct_dense, blr.hpp:62-86): diagonal tiles copied,
 * off-diagonal tiles expanded as (U X) Vt in the reference's order. `out` is a
 * device buffer (asynchronous on `stream`) when on_device, else a host buffer
 * (synchronous).
 */
lrb_status lrb_blr_reconstruct_dense(lrb_ctx* ctx, lrb_blr* m, double* out, int on_device,
                                     void* stream);

/* ------------------------------------------------------------ CUDA graphs */
/*
 * Capture every lrb_* launch issued on `stream` (a non-default stream)
 * between begin and end into a CUDA graph; replaying it issues the whole
 * sequence with one host call (no per-launch validation, tensor-map encoding
 * or driver overhead). Operand pointers are baked in at capture time.
 */
typedef struct lrb_graph lrb_graph;
lrb_status lrb_graph_begin(lrb_ctx* ctx, void* stream);
lrb_status lrb_graph_end(lrb_ctx* ctx, void* stream, lrb_graph** out);
lrb_status lrb_graph_launch(lrb_ctx* ctx, const lrb_graph* graph, void* stream);
lrb_status lrb_graph_destroy(lrb_ctx* ctx, lrb_graph* graph);
/* kernel launches one replay performs */
uint64_t lrb_graph_launches(const lrb_graph* graph);

/* ---------------------------------------------------- selector / planner */
typedef struct lrb_selection {
  int variant;        /* index into the variant table */
  int tile_m, tile_n; /* C tile per CTA (column-major view) */
  int tile_k;         /* k chunk per pipeline stage */
  int stages;         /* shared-memory pipeline depth */
  int threads;        /* threads per CTA (consumer warps + 1 TMA producer warp) */
  int ctas_per_sm;    /* design occupancy */
  int64_t tiles;      /* CTA tiles in the launch */
  int64_t grid;       /* persistent grid size */
  double intensity;   /* algorithmic flop / byte of the whole batch */
  int fp64_bound;     /* 1 if intensity >= measured FP64 ridge, else HBM-bound */
  char name[24];
} lrb_selection;

/*
 * Per-shape kernel selector (B200 analogue of make_packing_plan,
 * plan.hpp:66-100). ctx may be NULL (host-only: assumes 148 SMs). The choice
 * can be forced with lrb_set_variant_override or the LRB_VARIANT environment
 * variable (variant name), mirroring the reference's plan-override file
 * (plan.hpp:106-158).
 */
lrb_status lrb_select(const lrb_ctx* ctx, char order, char opA, char opB, int64_t m, int64_t n,
                      int64_t k, int64_t batch, lrb_selection* out);
int lrb_variant_count(void);
const char* lrb_variant_name(int variant);
int lrb_variant_from_name(const char* name); /* -1 if unknown */
lrb_status lrb_set_variant_override(lrb_ctx* ctx, int variant); /* -1 = automatic */
/* operand loader: -1 automatic (TMA tensor maps when the operands are 16-B
 * aligned with even leading dimensions / strides), 0 force the per-segment
 * bulk-copy loader, 1 TMA when eligible. Env LRB_LOADER=segment forces 0. */
lrb_status lrb_set_loader_override(lrb_ctx* ctx, int mode);

/*
 * Shard planner: split `batch` independent items into `nparts` contiguous
 * ranges, begin[0..nparts] (begin[0] = 0, begin[nparts] = batch). With
 * item_cost == NULL the split is the reference's contiguous fan-out
 * (per = ceil(batch / nparts); bench.hpp:69-75, kernels.hpp:274-276); with
 * costs, cuts are placed at equal cumulative cost. Host-only.
 */
lrb_status lrb_shard_plan(int64_t batch, const double* item_cost, int nparts, int64_t* begin);

/* algorithmic accounting of one item (beta = 0: 8(mk+kn+mn) bytes; beta = 1 adds mn) */
double lrb_item_flops(int64_t m, int64_t n, int64_t k);
double lrb_item_bytes(int64_t m, int64_t n, int64_t k, double beta);

/* ------------------------------------------------------- synthetic inputs */
/*
 * Fill `batch` column-major rows x cols matrices (leading dimension ld, item
 * stride `stride` elements) with lrb_uniform(seed, role, item_offset + i, elem)
 * from lrb_rng.h — bit-identical to the host generator.
 */
lrb_status lrb_fill_uniform(lrb_ctx* ctx, double* dst, int64_t rows, int64_t cols, int64_t ld,
                            int64_t stride, int64_t batch, uint64_t seed, uint32_t role,
                            int64_t item_offset, void* stream);
/* pointer-array form: host arrays of device pointers and per-item dims */
lrb_status lrb_fill_uniform_ptr(lrb_ctx* ctx, double* const* dst, const int64_t* rows,
                                const int64_t* cols, const int64_t* ld, int64_t batch,
                                uint64_t seed, uint32_t role, int64_t item_offset, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* LRB_H */
