// lrb_gemm.cuh — the batched FP64 GEMM kernel family (sm_100a).
//
// C_i = op(A_i) * op(B_i) + beta * C_i, column-major, beta in {0, 1}.
// Replaces the reference's per-item oracle loop nest
//   for i: for j: sum = accumulate ? c : 0; for p: sum += a[i,p] * b[p,j]
// (reference: proj/include/lrbatch/dense.hpp:43-56) over a batch.
//
// Structure (persistent CTAs):
//   * The CTA walks a flattened sequence of (tile, k-chunk) pairs: tiles
//     blockIdx.x, +gridDim.x, ...; each tile's k range in KB-wide chunks.
//   * Operands reach shared memory only through TMA. TMA=true (the fast
//     path): ONE cp.async.bulk.tensor.3d (SASS UTMALDG) per operand per stage
//     from a (rows, cols, batch) tensor map; the box is 4 elements wider than
//     the tile along its contiguous dimension, so the landed tile has a row
//     pitch == 4 (mod 16) doubles and the DMMA fragment loads are
//     bank-conflict free (64-bit loads are served per half-warp: lanes
//     (g, tq) g<4 hit pitch*tq + g, 16 distinct bank pairs). Ragged edges are
//     zero-filled by TMA. TMA=false (misaligned operands: odd ld, unaligned
//     base): one cp.async.bulk per contiguous column segment, or per-lane
//     plain loads where a segment is not 16-byte aligned/sized.
//   * The ring has STAGES slots, refilled in one of three forms:
//     - producer warp (ProdCfg, the 4-warp tiles): a fifth warp walks the
//       chunk sequence and issues each chunk as soon as the slot's empty
//       mbarrier completes; the computing warps only wait on full and arrive
//       on empty (r = 32 class 0.79-0.83 -> 0.92-0.95 of FP64 peak);
//     - producer warpgroup (ProdWgCfg, s96): the same with a whole producer
//       warpgroup whose registers go to the computing warpgroup (setmaxnreg);
//     - release counter (the 8-warp tiles, q64 with its TMA-store epilogue):
//       warp 0 issues chunks 0..STAGES-1; after a warp has consumed a slot it
//       bumps the slot's release counter, and the LAST warp to release it
//       issues the next chunk of the sequence into it.
//     Refills are issued in chunk order in every form.
//   * Each warp owns a WI x WJ sub-tile of C in registers as DMMA 8x8x4
//     fragments. The MMA computes C^T = op(B)^T op(A)^T so a lane's
//     accumulator pair is two consecutive ROWS of column-major C: the
//     epilogue is one 16-byte (32-byte for paired fragments) store per lane
//     and column. Write-bound strided tiles (beta = 0, k <= 16) instead stage
//     C in the consumed stage and leave through TMA stores (stage_c_tile).
//   * k is consumed in ascending order, 4 at a time by DMMA (each entry an
//     in-order FMA chain, probed bitwise on B200) and a scalar fma() tail, so
//     every C entry is exactly the reference's FMA chain.
// Shared-memory operand layouts (doubles):
//   K-rows   X_s[kk][o]  pitch = o_extent + 4   (op(A)=N, op(B)=T)
//   K-contig X_s[o][kk]  pitch = KB + 4         (op(A)=T, op(B)=N)
#pragma once

#include <cuda.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "lrb_device.cuh"

namespace lrb {

// ------------------------------------------------------------------ config
__host__ __device__ constexpr int round_up_c(int x, int m) { return (x + m - 1) / m * m; }
constexpr int kPad = 4;  // pitch == extent + 4 == 4 or 12 (mod 16) for extents multiple of 8

template <int WARPS_I_, int WARPS_J_, int WI_, int WJ_, int KB_, int STAGES_, int MINB_, bool A_T_,
          bool B_T_, bool TMA_>
struct GemmCfg {
  static constexpr int WARPS_I = WARPS_I_, WARPS_J = WARPS_J_, WI = WI_, WJ = WJ_;
  static constexpr int KB = KB_, STAGES = STAGES_, MINB = MINB_;
  static constexpr bool A_T = A_T_, B_T = B_T_, TMA = TMA_;
  static constexpr int MB = WARPS_I * WI, NB = WARPS_J * WJ;
  static constexpr int FI = WI / 8, FJ = WJ / 8;
  static constexpr int WARPS = WARPS_I * WARPS_J;
  static constexpr int THREADS = WARPS * 32;  // the computing warps
  // producer-warp form (ProdCfg): 0 here, all warps compute and refill
  static constexpr int PROD_WARPS = 0;
  static constexpr int LAUNCH_THREADS = THREADS;
  static constexpr int PROD_REGS = 0, MMA_REGS = 0;
  // operand pitches (doubles)
  static constexpr int PMA = MB + kPad;  // A K-rows  (op(A)=N): As[kk][i]
  static constexpr int PKA = KB + kPad;  // A K-contig (op(A)=T): As[i][kk]
  static constexpr int PNB = NB + kPad;  // B K-rows  (op(B)=T): Bs[kk][j]
  static constexpr int PKB = KB + kPad;  // B K-contig (op(B)=N): Bs[j][kk]
  // TMA boxes (inner = contiguous dim incl. pad, outer) == the landed layout
  static constexpr int A_BOX_IN = A_T ? PKA : PMA, A_BOX_OUT = A_T ? MB : KB;
  static constexpr int B_BOX_IN = B_T ? PNB : PKB, B_BOX_OUT = B_T ? KB : NB;
  static constexpr int A_BOX = A_BOX_IN * A_BOX_OUT, B_BOX = B_BOX_IN * B_BOX_OUT;
  static constexpr int A_ELEMS = round_up_c(A_BOX, 16);  // 128-B aligned sub-buffers
  static constexpr int B_ELEMS = round_up_c(B_BOX, 16);
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  // stages + full barriers + release counters + issue state
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * STAGE_ELEMS * 8 + size_t(STAGES) * 8 + size_t(STAGES) * 4 + 32;
  // TMA-store epilogue: the C tile is staged in the stage its last chunk just
  // used, as MB/16 boxes of 16 rows x NB columns in the 128-byte swizzle
  // (1024-byte aligned boxes), and written by the TMA engine
  static constexpr bool EPI_FITS = TMA_ && (MB % 16 == 0) && (MB * NB <= STAGE_ELEMS) &&
                                   (STAGE_ELEMS % 128 == 0) && (NB <= 256);
  static_assert(WI % 8 == 0 && WJ % 8 == 0, "warp tile must be a multiple of the 8x8 fragment");
  static_assert(KB % 4 == 0, "k chunk must be a multiple of the DMMA k (4)");
  static_assert(A_BOX_IN <= 256 && A_BOX_OUT <= 256 && B_BOX_IN <= 256 && B_BOX_OUT <= 256,
                "TMA box dimensions are limited to 256");

  // Fragment pairing: where the operand's tile dimension is contiguous in
  // shared memory (K-rows layouts), fragments (2p, 2p+1) take the adjacent
  // rows (2g, 2g+1): one conflict-free LDS.128 feeds two fragments, and (for
  // the i side) a lane's accumulators become 4 consecutive rows of C, stored
  // with one 32-byte st.global.v4 so each warp store covers whole 128-B lines.
  static constexpr bool PAIR_I = !A_T && (FI % 2 == 0);
  static constexpr bool PAIR_J = B_T && (FJ % 2 == 0);

  // in-tile row (i) of B-operand fragment fi / n-index g (loads)
  __device__ __forceinline__ static int load_row(int wi, int fi, int g) {
    return PAIR_I ? wi * WI + 16 * (fi >> 1) + 2 * g + (fi & 1) : wi * WI + 8 * fi + g;
  }
  // in-tile column (j) of A-operand fragment fj / row g (loads and accumulators)
  __device__ __forceinline__ static int load_col(int wj, int fj, int g) {
    return PAIR_J ? wj * WJ + 16 * (fj >> 1) + 2 * g + (fj & 1) : wj * WJ + 8 * fj + g;
  }
  // in-tile row of accumulator acc[.][fi][c] of lane quad tq
  __device__ __forceinline__ static int acc_row(int wi, int fi, int c, int tq) {
    return PAIR_I ? wi * WI + 16 * (fi >> 1) + 2 * (2 * tq + c) + (fi & 1)
                  : wi * WI + 8 * fi + 2 * tq + c;
  }

  // element offsets of op(A)(i, kk) and op(B)(kk, j) inside a stage
  __device__ __forceinline__ static int a_off(int i, int kk) {
    return A_T ? i * PKA + kk : kk * PMA + i;
  }
  __device__ __forceinline__ static int b_off(int kk, int j) {
    return B_T ? kk * PNB + j : j * PKB + kk;
  }
};

// Producer-warp form of a TMA configuration: one extra warp issues every
// refill behind per-slot empty mbarriers, so the computing warps only wait on
// full / arrive on empty per chunk (no release counter, tile decode or TMA
// issue on their path). With the TMA-store epilogue, warp 0 hands the slot
// back for all computing warps once the TMA engine has read the staged C.
template <class Base>
struct ProdCfg : Base {
  static constexpr int PROD_WARPS = 1;
  static constexpr int LAUNCH_THREADS = Base::THREADS + 32;
  static constexpr int PROD_REGS = 0, MMA_REGS = 0;  // no register hand-over
  // + the empty barriers (8-byte aligned after the release counters)
  static constexpr size_t SMEM_BYTES = Base::SMEM_BYTES + size_t(Base::STAGES) * 8 + 8;
  static_assert(Base::TMA, "the producer warp issues tensor-map loads only");
};

// Warpgroup-producer form for one computing warpgroup (4 warps) whose tiles
// need more registers than a plain fifth warp leaves (s96's 48 x 48 warp
// tiles): a whole producer warpgroup (one active warp) hands its registers
// to the computing warpgroup with setmaxnreg. Two CTAs per SM: 2 x 256
// threads at launch, then 128 x PR + 128 x MR = 32768 per CTA.
template <class Base, int PR, int MR>
struct ProdWgCfg : ProdCfg<Base> {
  static_assert(Base::WARPS == 4, "one computing warpgroup");
  static constexpr int PROD_WARPS = 4;
  static constexpr int LAUNCH_THREADS = Base::THREADS + 128;
  static constexpr int PROD_REGS = PR, MMA_REGS = MR;
};

// ---------------------------------------------------------------- problems
struct TileView {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int m, n, k;
  int i0, j0;
  const void* tmA;  // tensor maps (TMA path)
  const void* tmB;
  const void* tmC;  // C map for the TMA-store epilogue (strided problems)
  int za, zb, zc;   // batch coordinate inside the maps
  int zc2;          // 4-D C maps (BlrTileProblem): the tile-row coordinate
};

// Fixed-stride batch: item i at base + i * stride (the reference's
// LowRankBatch role arrays, low_rank.hpp:147-158).
struct StridedProblem {
  CUtensorMap tmA;  // (rows, cols, batch) maps of the stored operands
  CUtensorMap tmB;
  CUtensorMap tmC;  // (m, n, batch) map of C, box 16 x NB, 128-B swizzle (when c_tma)
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc, sA, sB, sC;
  int m, n, k;
  int tiles_i, tiles_per_item;
  int a_batched, b_batched;  // 0 when the stride is 0 (one matrix broadcast)
  int j_fastest;             // tile order inside an item: column tiles vary fastest
  int c_tma;                 // tmC is valid: beta = 0, k >= 1, C TMA-aligned
  int64_t num_tiles;

  static constexpr bool kDeferWait = false;
  // the A map and k coordinate of chunk k0 (two-source problems switch maps)
  __device__ __forceinline__ const void* a_src(const TileView& v, int k0, int* kc) const {
    *kc = k0;
    return v.tmA;
  }
  __device__ __forceinline__ bool tma_store() const { return c_tma != 0; }
  // TMA-store one staged 16-row box of C at tile rows (x, y) of item v
  __device__ __forceinline__ void store_box(const TileView& v, const double* src, int x,
                                            int y) const {
    tma_store_3d(v.tmC, src, x, y, v.zc);
  }

  template <int MB, int NB>
  __device__ __forceinline__ TileView tile(int64_t t) const {
    int64_t item;
    int r;
    if (num_tiles <= int64_t(UINT32_MAX)) {  // 32-bit divide on the common path
      const uint32_t tt = static_cast<uint32_t>(t), tpi = static_cast<uint32_t>(tiles_per_item);
      const uint32_t it = tt / tpi;
      item = it;
      r = static_cast<int>(tt - it * tpi);
    } else {
      item = t / tiles_per_item;
      r = static_cast<int>(t - item * tiles_per_item);
    }
    TileView v;
    v.A = A + item * sA;
    v.B = B + item * sB;
    v.C = C + item * sC;
    v.lda = lda;
    v.ldb = ldb;
    v.ldc = ldc;
    v.m = m;
    v.n = n;
    v.k = k;
    if (j_fastest) {
      const int tiles_j = tiles_per_item / tiles_i;
      v.i0 = (r / tiles_j) * MB;
      v.j0 = (r % tiles_j) * NB;
    } else {
      v.i0 = (r % tiles_i) * MB;
      v.j0 = (r / tiles_i) * NB;
    }
    v.tmA = &tmA;
    v.tmB = &tmB;
    v.tmC = &tmC;
    v.za = a_batched ? static_cast<int>(item) : 0;
    v.zb = b_batched ? static_cast<int>(item) : 0;
    v.zc = static_cast<int>(item);
    v.zc2 = 0;
    return v;
  }
  __device__ __forceinline__ int tile_k(int64_t) const { return k; }
};

// Pointer-array / variable-size batch: per-item descriptors (and, on the TMA
// path, a pair of 2-D tensor maps per item) plus a host-built tile list
// (item << 32 | ti << 16 | tj), largest k first.
struct ItemDesc {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int32_t m, n, k, pad;
};
static_assert(sizeof(ItemDesc) == 64, "ItemDesc is one 64-byte line");

struct PtrProblem {
  const ItemDesc* items;
  const uint64_t* tiles;
  const CUtensorMap* maps;  // 2 per item (A, B); null on the segment path
  int64_t num_tiles;

  static constexpr bool kDeferWait = false;
  __device__ __forceinline__ const void* a_src(const TileView& v, int k0, int* kc) const {
    *kc = k0;
    return v.tmA;
  }
  __device__ __forceinline__ bool tma_store() const { return false; }
  __device__ __forceinline__ void store_box(const TileView&, const double*, int, int) const {}

  template <int MB, int NB>
  __device__ __forceinline__ TileView tile(int64_t t) const {
    const uint64_t e = tiles[t];
    const uint32_t item = static_cast<uint32_t>(e >> 32);
    const ItemDesc d = items[item];
    TileView v;
    v.A = d.A;
    v.B = d.B;
    v.C = d.C;
    v.lda = d.lda;
    v.ldb = d.ldb;
    v.ldc = d.ldc;
    v.m = d.m;
    v.n = d.n;
    v.k = d.k;
    v.i0 = static_cast<int>((e >> 16) & 0xFFFF) * MB;
    v.j0 = static_cast<int>(e & 0xFFFF) * NB;
    v.tmA = maps ? &maps[2 * size_t(item)] : nullptr;
    v.tmB = maps ? &maps[2 * size_t(item) + 1] : nullptr;
    v.tmC = nullptr;
    v.za = 0;
    v.zb = 0;
    v.zc = 0;
    v.zc2 = 0;
    return v;
  }
  __device__ __forceinline__ int tile_k(int64_t t) const { return items[tiles[t] >> 32].k; }
};

// The off-diagonal tiles of a BLR matrix's dense reconstruction (reference
// blr.hpp:62-86): item q in the Vt-stacking order (column j, row i != j), C_q
// the b x b tile (i, j) of the n x n row-major output. In the column-major view
// C_q^T = Vt_q^T UX_q^T: A = Vt_q (b x r col-major, ld b), B = UX_q (r x b,
// ld r), both strided by q (3-D maps); C lives at out + i b n + j b with ld n.
// C leaves through a 4-D map (x, y, tile column j, tile row i) so the
// TMA-store epilogue covers every tile with one descriptor.
struct BlrTileProblem {
  CUtensorMap tmA;
  CUtensorMap tmB;
  CUtensorMap tmC;
  const double* A;  // Vt tiles, stacked by column
  const double* B;  // UX tiles, same order
  double* C;        // the n x n output
  int64_t n;
  int b, r, tiles;
  int tiles_i, tiles_per_item;
  int c_tma;
  int64_t num_tiles;

  static constexpr bool kDeferWait = false;
  __device__ __forceinline__ const void* a_src(const TileView& v, int k0, int* kc) const {
    *kc = k0;
    return v.tmA;
  }
  __device__ __forceinline__ bool tma_store() const { return c_tma != 0; }
  __device__ __forceinline__ void store_box(const TileView& v, const double* src, int x,
                                            int y) const {
    tma_store_4d(v.tmC, src, x, y, v.zc, v.zc2);
  }
  template <int MB, int NB>
  __device__ __forceinline__ TileView tile(int64_t t) const {
    const uint32_t tt = static_cast<uint32_t>(t), tpi = static_cast<uint32_t>(tiles_per_item);
    const uint32_t q = tt / tpi;
    const int rr = static_cast<int>(tt - q * tpi);
    const int j = int(q) / (tiles - 1), ip = int(q) - j * (tiles - 1);
    const int i = ip < j ? ip : ip + 1;
    TileView v;
    v.A = A + int64_t(q) * b * r;
    v.B = B + int64_t(q) * r * b;
    v.C = C + int64_t(i) * b * n + int64_t(j) * b;
    v.lda = b;
    v.ldb = r;
    v.ldc = n;
    v.m = b;
    v.n = b;
    v.k = r;
    v.i0 = (rr % tiles_i) * MB;
    v.j0 = (rr / tiles_i) * NB;
    v.tmA = &tmA;
    v.tmB = &tmB;
    v.tmC = &tmC;
    v.za = int(q);
    v.zb = int(q);
    v.zc = j;
    v.zc2 = i;
    return v;
  }
  __device__ __forceinline__ int tile_k(int64_t) const { return r; }
};

// The BLR matvec's row step y_i = [D_i | U_i*] [rhs_i; Z_i*] (lrb_blr.cu) in
// the column-major view y_i^T = [rhs_i^T | Z_i^T] [D_i | U_i*]^T: m = nrhs,
// n = b, k = b + (T-1) r. The A operand has two sources split at k = kb (= b,
// a multiple of the chunk depth): rhs_i (an input) for k < kb, and Z_i (the
// coupling kernel's output) beyond. The kernel therefore starts on the D_i
// rhs_i part while the coupling kernel still runs, and the issuing lane
// executes griddepcontrol.wait before the first chunk that reads Z.
struct BlrRowProblem {
  CUtensorMap tmA;   // rhs: (nrhs, b, T), item stride b nrhs
  CUtensorMap tmA2;  // Z: (nrhs, K, T), item stride pitch nrhs (rows b.. of rz)
  CUtensorMap tmB;   // [D_i | U_i*]: (pitch, b, T) column-major view
  double* C;         // y: nrhs x b per item (column-major view), ld nrhs
  int m, n, k, kb;
  int tiles_i, tiles_per_item;
  int64_t num_tiles;

  static constexpr bool kDeferWait = true;
  __device__ __forceinline__ const void* a_src(const TileView&, int k0, int* kc) const {
    if (k0 < kb) {
      *kc = k0;
      return &tmA;
    }
    pdl_wait();
    *kc = k0 - kb;
    return &tmA2;
  }
  __device__ __forceinline__ bool tma_store() const { return false; }
  __device__ __forceinline__ void store_box(const TileView&, const double*, int, int) const {}
  template <int MB, int NB>
  __device__ __forceinline__ TileView tile(int64_t t) const {
    const uint32_t tt = static_cast<uint32_t>(t), tpi = static_cast<uint32_t>(tiles_per_item);
    const uint32_t item = tt / tpi;
    const int rr = static_cast<int>(tt - item * tpi);
    TileView v;
    v.A = nullptr;  // TMA only
    v.B = nullptr;
    v.C = C + int64_t(item) * m * n;
    v.lda = m;
    v.ldb = k;
    v.ldc = m;
    v.m = m;
    v.n = n;
    v.k = k;
    v.i0 = (rr % tiles_i) * MB;
    v.j0 = (rr / tiles_i) * NB;
    v.tmA = &tmA;
    v.tmB = &tmB;
    v.tmC = nullptr;
    v.za = int(item);
    v.zb = int(item);
    v.zc = int(item);
    v.zc2 = 0;
    return v;
  }
  __device__ __forceinline__ int tile_k(int64_t) const { return k; }
};

// next chunk to issue, shared by the CTA's warps
struct IssueState {
  long long t;
  int k0;
  int pad;
};

// ------------------------------------------------------------------ kernel
template <class Problem>
__device__ __forceinline__ int64_t skip_empty_tiles(const Problem& prob, int64_t t) {
  while (t < prob.num_tiles && prob.tile_k(t) == 0) t += gridDim.x;
  return t;
}

// Issue the chunk described by *st into `stage` (whole warp), then advance *st.
// Issue the TMA loads of chunk (v, k0) into `stage` (one lane).
template <class Cfg, class Problem>
__device__ __forceinline__ void issue_tma(const Problem& prob, const TileView& v, int k0,
                                          double* As, double* Bs, uint64_t* full, int stage,
                                          int flags) {
  constexpr int MB = Cfg::MB, NB = Cfg::NB;
  // An operand is streamed once when one column (A) / row (B) tile covers
  // C, else reused by the neighbouring tiles (evict-last). Single-use
  // streams still load evict-normal, not evict-first: every box reads
  // kPad elements past the tile for its pitch — the next chunk's first
  // k-columns (k-contiguous boxes) or the neighbouring tile's first rows —
  // which must still be in L2 when that chunk or tile is loaded (measured:
  // r = 8/16 sweeps 0.87-0.99 -> 0.95-1.04 of HBM)
  uint64_t pol_a = (v.n <= NB) ? policy_evict_normal() : policy_evict_last();
  uint64_t pol_b = (v.m <= MB) ? policy_evict_normal() : policy_evict_last();
  if (flags & 32) pol_a = pol_b = policy_evict_normal();  // debug probes
  if (flags & 128) pol_a = pol_b = policy_evict_first();
  mbar_arrive_expect_tx(&full[stage], uint32_t(Cfg::A_BOX + Cfg::B_BOX) * 8u);
  int ka;
  const void* map_a = prob.a_src(v, k0, &ka);
  if (Cfg::A_T)
    tma_load_3d(As, map_a, ka, v.i0, v.za, &full[stage], pol_a);
  else
    tma_load_3d(As, map_a, v.i0, ka, v.za, &full[stage], pol_a);
  if (Cfg::B_T)
    tma_load_3d(Bs, v.tmB, v.j0, k0, v.zb, &full[stage], pol_b);
  else
    tma_load_3d(Bs, v.tmB, k0, v.j0, v.zb, &full[stage], pol_b);
}

template <class Cfg, class Problem>
__device__ __forceinline__ void issue_chunk(const Problem& prob, double* smem, uint64_t* full,
                                            IssueState* st, int stage, int lane, int flags) {
  constexpr int MB = Cfg::MB, NB = Cfg::NB, KB = Cfg::KB;
  // lane 0 (which synchronised with the previous issuer through the release
  // counter) reads the shared state and broadcasts it
  long long t_ll = 0;
  int k0 = 0;
  if (lane == 0) {
    t_ll = st->t;
    k0 = st->k0;
  }
  const int64_t t = __shfl_sync(0xffffffffu, t_ll, 0);
  k0 = __shfl_sync(0xffffffffu, k0, 0);
  if (t >= prob.num_tiles) return;  // sequence exhausted (uniform across the warp)
  const TileView v = prob.template tile<MB, NB>(t);
  double* As = smem + size_t(stage) * Cfg::STAGE_ELEMS;
  double* Bs = As + Cfg::A_ELEMS;
  // order this CTA's generic-proxy reads of the slot before the async-proxy refill
  fence_proxy_async_smem();
  if constexpr (Cfg::TMA) {
    if (lane == 0) issue_tma<Cfg>(prob, v, k0, As, Bs, full, stage, flags);
  } else {
    const int ivalid = min(MB, v.m - v.i0);
    const int jvalid = min(NB, v.n - v.j0);
    const int kvalid = min(KB, v.k - k0);
    const uint64_t pol_a = (v.n <= NB) ? policy_evict_first() : policy_evict_last();
    const uint64_t pol_b = (v.m <= MB) ? policy_evict_first() : policy_evict_last();
    const int seg_a = Cfg::A_T ? ivalid : kvalid;
    const int seg_b = Cfg::B_T ? kvalid : jvalid;
    uint32_t bytes = 0;
#pragma unroll 1
    for (int s = lane; s < seg_a + seg_b; s += 32) {
      const double* src;
      double* dst;
      int len;
      uint64_t pol;
      if (s < seg_a) {
        if (Cfg::A_T) {
          src = v.A + k0 + int64_t(v.i0 + s) * v.lda;
          dst = As + s * Cfg::PKA;
          len = kvalid;
        } else {
          src = v.A + v.i0 + int64_t(k0 + s) * v.lda;
          dst = As + s * Cfg::PMA;
          len = ivalid;
        }
        pol = pol_a;
      } else {
        const int q = s - seg_a;
        if (Cfg::B_T) {
          src = v.B + v.j0 + int64_t(k0 + q) * v.ldb;
          dst = Bs + q * Cfg::PNB;
          len = jvalid;
        } else {
          src = v.B + k0 + int64_t(v.j0 + q) * v.ldb;
          dst = Bs + q * Cfg::PKB;
          len = kvalid;
        }
        pol = pol_b;
      }
      const uint32_t nb = uint32_t(len) * 8u;
      if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((nb & 15) == 0)) {
        bulk_g2s(dst, src, nb, &full[stage], pol);
        bytes += nb;
      } else {
#pragma unroll 4
        for (int e = 0; e < len; ++e) dst[e] = __ldg(src + e);
      }
    }
    bytes = __reduce_add_sync(0xffffffffu, bytes);
    __syncwarp();
    if (lane == 0) {
      if (bytes)
        mbar_arrive_expect_tx(&full[stage], bytes);
      else
        mbar_arrive(&full[stage]);
    }
  }
  if (lane == 0) {  // advance the sequence
    int nk0 = k0 + KB;
    int64_t nt = t;
    if (nk0 >= v.k) {
      nk0 = 0;
      nt = skip_empty_tiles(prob, t + gridDim.x);
    }
    st->t = nt;
    st->k0 = nk0;
  }
  __syncwarp();
}

template <class Cfg>
__device__ __forceinline__ void mma_kstep(double (&acc)[Cfg::FJ][Cfg::FI][2], const double* As,
                                          const double* Bs, int wi, int wj, int g, int kk) {
  double af[Cfg::FJ], bf[Cfg::FI];
  if constexpr (Cfg::PAIR_J) {
#pragma unroll
    for (int q = 0; q < Cfg::FJ / 2; ++q) {
      const double2 v =
          *reinterpret_cast<const double2*>(&Bs[Cfg::b_off(kk, Cfg::load_col(wj, 2 * q, g))]);
      af[2 * q] = v.x;
      af[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int fj = 0; fj < Cfg::FJ; ++fj) af[fj] = Bs[Cfg::b_off(kk, Cfg::load_col(wj, fj, g))];
  }
  if constexpr (Cfg::PAIR_I) {
#pragma unroll
    for (int p = 0; p < Cfg::FI / 2; ++p) {
      const double2 v =
          *reinterpret_cast<const double2*>(&As[Cfg::a_off(Cfg::load_row(wi, 2 * p, g), kk)]);
      bf[2 * p] = v.x;
      bf[2 * p + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int fi = 0; fi < Cfg::FI; ++fi) bf[fi] = As[Cfg::a_off(Cfg::load_row(wi, fi, g), kk)];
  }
#pragma unroll
  for (int fj = 0; fj < Cfg::FJ; ++fj)
#pragma unroll
    for (int fi = 0; fi < Cfg::FI; ++fi) dmma_8x8x4(acc[fj][fi][0], acc[fj][fi][1], af[fj], bf[fi]);
}

// Stage a warp's accumulators as C-tile boxes for the TMA store: box q holds
// tile rows 16q..16q+15 of all NB columns, column j a 128-byte row with its
// 16-byte chunks XOR-swizzled by (j & 7) (CU_TENSOR_MAP_SWIZZLE_128B).
template <class Cfg>
__device__ __forceinline__ int c_stage_off(int i, int j) {
  const int q = i >> 4, il = i & 15;
  return q * 16 * Cfg::NB + j * 16 + ((((il >> 1) ^ (j & 7))) << 1) + (il & 1);
}

template <class Cfg>
__device__ __forceinline__ void stage_c_tile(double* cs, const double (&acc)[Cfg::FJ][Cfg::FI][2],
                                             int wi, int wj, int g, int tq) {
#pragma unroll
  for (int fj = 0; fj < Cfg::FJ; ++fj) {
    const int j = Cfg::load_col(wj, fj, g);
    if constexpr (Cfg::PAIR_I) {
#pragma unroll
      for (int p = 0; p < Cfg::FI / 2; ++p) {
        const int i = Cfg::acc_row(wi, 2 * p, 0, tq);  // rows i .. i+3, i % 4 == 0
        sts128(cs + c_stage_off<Cfg>(i, j), acc[fj][2 * p][0], acc[fj][2 * p + 1][0]);
        sts128(cs + c_stage_off<Cfg>(i + 2, j), acc[fj][2 * p][1], acc[fj][2 * p + 1][1]);
      }
    } else {
#pragma unroll
      for (int fi = 0; fi < Cfg::FI; ++fi) {
        const int i = Cfg::acc_row(wi, fi, 0, tq);  // rows i, i+1 (i even)
        sts128(cs + c_stage_off<Cfg>(i, j), acc[fj][fi][0], acc[fj][fi][1]);
      }
    }
  }
}

template <class Cfg, class Problem>
__global__ void __launch_bounds__(Cfg::LAUNCH_THREADS, Cfg::MINB)
    lrb_gemm_kernel(const __grid_constant__ Problem prob, const int flags) {
  static_assert(Cfg::WARPS % 4 == 0, "warps per CTA must fill all four SM sub-partitions");
  if constexpr (Problem::kDeferWait)
    pdl_trigger();  // the problem waits before its first dependent load
  else
    pdl_entry();
  // flags bit 0: beta = 1 (accumulate into C); debug probes (LRB_DEBUG_FLAGS,
  // never set by the library itself): bit 1 skips the epilogue stores, bit 3
  // uses default-policy instead of streaming stores, bit 4 stops refilling the
  // ring after the prologue (MMAs on stale data; bit 2 is host-side)
  const int beta_one = flags & 1;
  // C leaves through the TMA engine from shared memory (strided problems with
  // beta = 0 and a TMA-aligned C, variants whose C tile fits one stage)
  const bool epi_tma = Cfg::EPI_FITS && prob.tma_store();
  constexpr int MB = Cfg::MB, NB = Cfg::NB, KB = Cfg::KB, STAGES = Cfg::STAGES;
  constexpr int FI = Cfg::FI, FJ = Cfg::FJ;
  // dynamic shared memory starts 1024-B aligned (no static shared memory);
  // keep every pointer derived from this array so loads stay LDS
  extern __shared__ __align__(1024) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * Cfg::STAGE_ELEMS);
  IssueState* st = reinterpret_cast<IssueState*>(full + STAGES);
  int* released = reinterpret_cast<int*>(st + 1);
  // producer form: per-slot empty barriers after the release counters
  uint64_t* empty = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(released + STAGES) + 7) & ~uintptr_t(7));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
      if constexpr (Cfg::PROD_WARPS > 0) mbar_init(&empty[s], Cfg::WARPS);
    }
    st->t = skip_empty_tiles(prob, int64_t(blockIdx.x));
    st->k0 = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (Cfg::PROD_WARPS > 0) {
    if (warp >= Cfg::WARPS) {
      // warpgroup form: hand the producer warpgroup's registers to the
      // computing warpgroup
      if constexpr (Cfg::PROD_REGS > 0)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::PROD_REGS));
      // the producer: the CTA's (tile, k-chunk) sequence in order, each
      // chunk into slot q % STAGES once the computing warps have released it
      if (warp == Cfg::WARPS && lane == 0) {
        int64_t t = skip_empty_tiles(prob, int64_t(blockIdx.x));
        int k0 = 0;
        int stage = 0;
        uint32_t phase = 0;
        int64_t q = 0;
#pragma unroll 1
        while (t < prob.num_tiles) {
          const TileView v = prob.template tile<MB, NB>(t);
          if (q >= STAGES) mbar_wait(&empty[stage], phase ^ 1);
          fence_proxy_async_smem();
          double* As = smem + size_t(stage) * Cfg::STAGE_ELEMS;
          issue_tma<Cfg>(prob, v, k0, As, As + Cfg::A_ELEMS, full, stage, flags);
          k0 += KB;
          if (k0 >= v.k) {
            k0 = 0;
            t = skip_empty_tiles(prob, t + gridDim.x);
          }
          ++q;
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      return;
    }
    if constexpr (Cfg::MMA_REGS > 0)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::MMA_REGS));
  } else {
    if (warp == 0) {
#pragma unroll 1
      for (int s = 0; s < STAGES; ++s) issue_chunk<Cfg>(prob, smem, full, st, s, lane, flags);
    }
  }

  const int wi = warp % Cfg::WARPS_I;
  const int wj = warp / Cfg::WARPS_I;
  const int g = lane >> 2;
  const int tq = lane & 3;
  // in-tile coordinates of this lane's fragments: Cfg::load_row / load_col /
  // acc_row (accumulator acc[fj][fi][c] is C(acc_row(fi, c), load_col(fj)))

  int stage = 0;
  uint32_t phase = 0;
  int consumed = 0;  // debug probe bit 4: after the prologue, compute on stale data
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < prob.num_tiles; t += gridDim.x) {
    const TileView v = prob.template tile<MB, NB>(t);
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(v.C) & 15) == 0) && ((v.ldc & 1) == 0);
    const bool vec4_ok = ((reinterpret_cast<uintptr_t>(v.C) & 31) == 0) && ((v.ldc & 3) == 0);

    double acc[FJ][FI][2];
#pragma unroll
    for (int fj = 0; fj < FJ; ++fj)
#pragma unroll
      for (int fi = 0; fi < FI; ++fi) acc[fj][fi][0] = acc[fj][fi][1] = 0.0;
    if (beta_one) {
#pragma unroll
      for (int fj = 0; fj < FJ; ++fj) {
        const int j = v.j0 + Cfg::load_col(wj, fj, g);
        if (j < v.n) {
          const double* cp = v.C + int64_t(j) * v.ldc;
#pragma unroll
          for (int fi = 0; fi < FI; ++fi)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int i = v.i0 + Cfg::acc_row(wi, fi, c, tq);
              if (i < v.m) acc[fj][fi][c] = cp[i];
            }
        }
      }
    }

#pragma unroll 1
    for (int k0 = 0; k0 < v.k; k0 += KB) {
      const int kvalid = min(KB, v.k - k0);
      if (!(flags & 16) || consumed < STAGES) mbar_wait(&full[stage], phase);
      ++consumed;
      const double* As = smem + size_t(stage) * Cfg::STAGE_ELEMS;
      const double* Bs = As + Cfg::A_ELEMS;
      if (kvalid == KB) {
#pragma unroll
        for (int kq = 0; kq < KB / 4; ++kq) mma_kstep<Cfg>(acc, As, Bs, wi, wj, g, kq * 4 + tq);
      } else {
        const int nq = kvalid >> 2;
#pragma unroll 1
        for (int kq = 0; kq < nq; ++kq) mma_kstep<Cfg>(acc, As, Bs, wi, wj, g, kq * 4 + tq);
        // scalar tail keeps the in-order FMA chain for k % 4 != 0
#pragma unroll 1
        for (int kk = nq * 4; kk < kvalid; ++kk) {
#pragma unroll
          for (int fj = 0; fj < FJ; ++fj) {
            const double bv = Bs[Cfg::b_off(kk, Cfg::load_col(wj, fj, g))];
#pragma unroll
            for (int fi = 0; fi < FI; ++fi)
#pragma unroll
              for (int c = 0; c < 2; ++c)
                acc[fj][fi][c] =
                    fma(As[Cfg::a_off(Cfg::acc_row(wi, fi, c, tq), kk)], bv, acc[fj][fi][c]);
          }
        }
      }
      if (epi_tma && k0 + KB >= v.k) {
        // TMA-store epilogue: once every warp is done with the slot, stage C
        // there (swizzled), hand it to the TMA engine, and refill the slot as
        // soon as the engine has read it. The named barriers also order the
        // issue state between this issuer and the previous one.
        named_barrier_sync(1, Cfg::THREADS);
        double* cs = smem + size_t(stage) * Cfg::STAGE_ELEMS;
        stage_c_tile<Cfg>(cs, acc, wi, wj, g, tq);
        fence_proxy_async_shared_cta();
        named_barrier_sync(1, Cfg::THREADS);
        if (warp == 0) {
          if (lane == 0) {
            if (!(flags & 2)) {
#pragma unroll 1
              for (int q = 0; q < MB / 16; ++q)
                if (v.i0 + 16 * q < v.m)
                  prob.store_box(v, cs + q * 16 * NB, v.i0 + 16 * q, v.j0);
            }
            bulk_commit_group();
            bulk_wait_group_read0();
          }
          __syncwarp();
          if constexpr (Cfg::PROD_WARPS > 0) {
            if (lane == 0) mbar_arrive_cnt(&empty[stage], Cfg::WARPS);
          } else if (!(flags & 16)) {
            issue_chunk<Cfg>(prob, smem, full, st, stage, lane, flags);
          }
        }
      } else if constexpr (Cfg::PROD_WARPS > 0) {
        // hand the slot back to the producer
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      } else {
        // release the slot; the last warp out refills it with the next chunk
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          // acq_rel: orders this warp's reads of the slot before the count, and
          // lets the last warp see the issue state the previous issuer wrote
          last = (atom_add_acq_rel_cta(&released[stage], 1) == Cfg::WARPS - 1);
          if (last) released[stage] = 0;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last && !(flags & 16)) issue_chunk<Cfg>(prob, smem, full, st, stage, lane, flags);
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    if (epi_tma) continue;  // C was stored from shared memory at the last chunk
    // epilogue: consecutive rows of one column of C per lane — 4 rows (one
    // 32-B store) for paired fragments, else 2 rows (one 16-B store)
    if (flags & 2) continue;
#pragma unroll
    for (int fj = 0; fj < FJ; ++fj) {
      const int j = v.j0 + Cfg::load_col(wj, fj, g);
      if (j < v.n) {
        double* cp = v.C + int64_t(j) * v.ldc;
        if constexpr (Cfg::PAIR_I) {
#pragma unroll
          for (int p = 0; p < FI / 2; ++p) {
            const int i = v.i0 + Cfg::acc_row(wi, 2 * p, 0, tq);  // rows i .. i+3
            const double r0 = acc[fj][2 * p][0], r1 = acc[fj][2 * p + 1][0];
            const double r2 = acc[fj][2 * p][1], r3 = acc[fj][2 * p + 1][1];
            if (vec4_ok && i + 3 < v.m) {
              if (flags & 8)
                st_global_v4_wb(cp + i, r0, r1, r2, r3);
              else
                st_global_v4(cp + i, r0, r1, r2, r3);
            } else {
              if (i < v.m) st_global_cs(cp + i, r0);
              if (i + 1 < v.m) st_global_cs(cp + i + 1, r1);
              if (i + 2 < v.m) st_global_cs(cp + i + 2, r2);
              if (i + 3 < v.m) st_global_cs(cp + i + 3, r3);
            }
          }
        } else {
#pragma unroll
          for (int fi = 0; fi < FI; ++fi) {
            const int i = v.i0 + Cfg::acc_row(wi, fi, 0, tq);  // rows i, i+1
            if (vec_ok && i + 1 < v.m) {
              st_global_v2(cp + i, acc[fj][fi][0], acc[fj][fi][1]);
            } else {
              if (i < v.m) st_global_cs(cp + i, acc[fj][fi][0]);
              if (i + 1 < v.m) st_global_cs(cp + i + 1, acc[fj][fi][1]);
            }
          }
        }
      }
    }
  }
  // the TMA stores this CTA issued must land before the grid completes
  if (epi_tma && threadIdx.x == 0) bulk_wait_group0();
}

// ------------------------------------------------------------------ launch
struct LaunchInfo {
  int64_t grid;
  int occupancy;
};

template <class Cfg, class Problem>
cudaError_t launch_gemm(const Problem& prob, int beta_one, int device, int sm_count,
                        cudaStream_t stream, LaunchInfo* info) {
  auto kern = lrb_gemm_kernel<Cfg, Problem>;
  // per-device one-time attribute + occupancy query
  static int occ_cache[64] = {0};
  int occ = (device >= 0 && device < 64) ? occ_cache[device] : 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::SMEM_BYTES));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::LAUNCH_THREADS,
                                                      Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (device >= 0 && device < 64) occ_cache[device] = occ;
  }
  int64_t grid = int64_t(sm_count) * occ;
  if (prob.num_tiles < grid) grid = prob.num_tiles;
  if (info) {
    info->grid = grid;
    info->occupancy = occ;
  }
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(Cfg::LAUNCH_THREADS), Cfg::SMEM_BYTES,
                    stream, prob, beta_one);
}

}  // namespace lrb
