// lrb_variants.h — the kernel variant table shared by the selector (host) and
// the per-variant instantiation units (device).
//
// A variant fixes the CTA tile of C (column-major view): MB = WARPS_I * WI rows
// by NB = WARPS_J * WJ columns, computed by WARPS_I * WARPS_J warps (warp tile
// WI rows x WJ columns, DMMA 8x8x4 fragments) fed through a STAGES-deep
// shared-memory ring of KB-wide k chunks that the warps refill themselves
// (lrb_gemm.cuh), MINB CTAs per SM.
//
//   n*  : tall-skinny C (dense b x b times a b x r basis, r <= 64): the BLR
//         diagonal shape (reference blr.hpp:149-153) in column-major — HBM
//         streaming of the b x b block, two CTAs per SM.
//   m*  : short-wide C, the same product issued row-major (swapped operands).
//   sq  : 128 x 128 tiles for the low-rank expansion U * V^T (blr.hpp:75-78),
//         write-dominated and at the FP64 ridge.
//   n64 : 128 x 64 tiles at two CTAs per SM (r in 57..64).
//   q64 : 64 x 64 tiles at three CTAs per SM — the general-shape choice (the
//         low-rank expansion U * V^T, blr.hpp:75-78): more independent CTAs
//         overlap one CTA's epilogue and operand wait with the others' MMAs.
//   n64s4 : KB = 16 alternative kept for the selector sweep.
//   n16t : 32-row tiles at seven CTAs per SM for small skinny batches (cfg1;
//         seven with the producer warp: 2048 tiles in 1.98 waves).
//   n16h : 64-row tiles, sweep candidate.
//   m8t, m16t : 32-column tiles at five CTAs per SM, the m* shapes of small
//         batches (the BLR matvec's per-row launches: 64 items of 8 x 512).
//   t64 : 128 x 64 tiles, 64 x 32 per warp (256 DMMAs per k-chunk instead of
//         128), two CTAs per SM: general shapes with a long inner dimension
//         (k >= 128), where the per-tile overhead then amortises (the
//         low-rank product's r = 128 GEMMs: 0.86 -> 0.94 of FP64 peak).
//   m8k64, m16k64 : 64-column tiles with KB = 64 for the short-wide class. The
//         row-major drop-in stores the big block contiguous along k, so its
//         TMA box is NB segments of KB doubles: 512-byte instead of 256-byte
//         segments raise the r = 8/16 row-major sweep from 0.75-0.89 to
//         0.84-0.96 of HBM.
//   s96 : 96 x 96 tiles (48 x 48 per warp), two CTAs per SM: outputs whose
//         sides are (multiples of) 96, where 64- and 128-wide tiles pad 96 to
//         128 (the paper's rank-96 low-rank products: 0.48 -> 0.93).
//   n24, n40, n48, n56 : intermediate widths so a variable-rank batch
//         (cfg4, r_i in 8..64) wastes less than one 8-column fragment; all
//         four warps 32 rows tall (n48 / n56: 32 x 48 / 32 x 56 warp tiles).
//   q64p : q64 with a producer warp (lrb_dispatch.cuh VariantProd), for
//         general shapes with k > 16; q64 itself keeps the TMA-store
//         epilogue's synchronous slot hand-back for the write-bound k <= 16.
//   q64q : q64p with a 3-stage ring at two CTAs per SM, for k >= 256 (the
//         low-rank r = 64 product's 64 x 64 x b GEMM: +5-6%).
// (Measured and dropped: n32 with 16-deep chunks in a 3-stage ring at three
// CTAs per SM, 0.80-0.87 of the r = 32 class's roofline against n32's
// 0.88-0.95 on the same box.)
// The 4-warp variants run a producer warp on their TMA path (VariantProd):
// the computing warps then only wait on full / arrive on empty per chunk.
#pragma once

//            id  name  WARPS_I WARPS_J WI  WJ  KB  STAGES MINB
#define LRB_VARIANT_LIST(X)          \
  X(0, n8, 4, 1, 32, 8, 32, 2, 2)    \
  X(1, n16, 4, 1, 32, 16, 32, 2, 2)  \
  X(2, n32, 4, 1, 32, 32, 32, 2, 2)  \
  X(3, n64, 4, 2, 32, 32, 32, 2, 2)  \
  X(4, sq, 2, 4, 64, 32, 32, 3, 1)   \
  X(5, m8, 1, 4, 8, 32, 32, 2, 2)    \
  X(6, m16, 1, 4, 16, 32, 32, 2, 2)  \
  X(7, m32, 1, 4, 32, 32, 32, 2, 2)  \
  X(8, m64, 2, 4, 32, 32, 32, 2, 2)  \
  X(9, n24, 4, 1, 32, 24, 32, 2, 2)  \
  X(10, n40, 4, 1, 32, 40, 32, 2, 2) \
  X(11, n48, 4, 1, 32, 48, 32, 2, 2) \
  X(12, n56, 4, 1, 32, 56, 32, 2, 2) \
  X(13, q64, 2, 2, 32, 32, 32, 2, 3) \
  X(14, n64s4, 4, 2, 32, 32, 16, 4, 2) \
  X(15, n16t, 4, 1, 8, 16, 32, 2, 7)   \
  X(16, n16h, 4, 1, 16, 16, 32, 2, 4)  \
  X(17, m8t, 1, 4, 8, 8, 32, 2, 5)     \
  X(18, m16t, 1, 4, 16, 8, 32, 2, 5)   \
  X(19, t64, 2, 2, 64, 32, 32, 2, 2)   \
  X(20, s96, 2, 2, 48, 48, 32, 2, 2)   \
  X(21, m16k64, 1, 4, 16, 16, 64, 2, 2) \
  X(22, m8k64, 1, 4, 8, 16, 64, 2, 2)  \
  X(23, q64p, 2, 2, 32, 32, 32, 2, 3) \
  X(24, q64q, 2, 2, 32, 32, 32, 3, 2)

#define LRB_NUM_VARIANTS 25

enum {
  LRB_V_N8 = 0,
  LRB_V_N16 = 1,
  LRB_V_N32 = 2,
  LRB_V_N64 = 3,
  LRB_V_SQ = 4,
  LRB_V_M8 = 5,
  LRB_V_M16 = 6,
  LRB_V_M32 = 7,
  LRB_V_M64 = 8,
  LRB_V_N24 = 9,
  LRB_V_N40 = 10,
  LRB_V_N48 = 11,
  LRB_V_N56 = 12,
  LRB_V_Q64 = 13,
  LRB_V_N64S4 = 14,
  LRB_V_N16T = 15,
  LRB_V_N16H = 16,
  LRB_V_M8T = 17,
  LRB_V_M16T = 18,
  LRB_V_T64 = 19,
  LRB_V_S96 = 20,
  LRB_V_M16K64 = 21,
  LRB_V_M8K64 = 22,
  LRB_V_Q64P = 23,
  LRB_V_Q64Q = 24
};
