// lrb_blr_recon.cu — (U X) Vt expansions as ONE write-streaming kernel, in
// two addressing modes:
//   * the off-diagonal tiles of BlrMatrix::reconstruct_dense (reference
//     blr.hpp:62-86: out tile (i, j) = dense_gemm_naive(dense_gemm_naive(U_ij,
//     X_ij), Vt_ij)), U rows read from the [D_i | U_i*] row panel;
//   * the batched low-rank expansion out_q = (U_q X_q) Vt_q
//     (lrb_lowrank_expand, the same per-tile product over LowRankOperands).
//
// The output is ~90 % of the bytes, so the kernel is built around keeping the
// TMA store stream full:
//   * unit = (item q, 64-row block, 256-column half): a producer warp lands
//     the half's Vt_q (two 3-D boxes of 128 + 4 columns x r rows), the
//     block's U_q rows (one box of r + 4 columns x 64 rows) and X_q (one bulk
//     copy per row, padded) into a 2-slot ring;
//   * eight computing warps (a 16 x 32 quarter-strip each) form UX = U X on
//     DMMA (rounded, the reference's first product) in registers, then
//     each 64 x 64 block of (UX) Vt on DMMA, k ascending — both chains as the
//     reference orders them, so results are bitwise the FMA-chain oracle;
//   * each warp stages its 16 x 32 part of two 64 x 64 output blocks in the
//     128-byte swizzle and hands them to the TMA engine itself (four 16 x 16
//     boxes, one proxy fence); two staging pairs per warp alternate, so the
//     warps never meet at a barrier and one pair per warp is in flight while
//     the next is computed.
// The BLR diagonal tiles are copied by blr_diag_kernel (lrb_blr.cu), which
// runs beside this kernel (one CTA per SM each; disjoint outputs).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "lrb_device.cuh"
#include "lrb_internal.h"

namespace lrb {

bool encode_operand(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                    int64_t stride, int64_t zdim, int box_in, int box_out);
bool encode_c_map(CUtensorMap* map, double* C, int64_t m, int64_t n, int64_t ldc, int64_t sC,
                  int64_t batch, int nb);

namespace {

constexpr int kRPad = 4;
constexpr int kRWarps = 8;
constexpr int kRThreads = kRWarps * 32 + 32;  // + the producer warp
constexpr int kRHalf = 256;                 // output columns per unit
constexpr int kRBox = 128;                  // Vt box columns (+ kRPad)
constexpr int kXPad = 0;                    // X lands unpadded by ONE bulk copy (a copy per padded row
                                            // was 8-16 tiny TMA ops per unit beside the store stream)
constexpr int kStageBufs = 4;                  // per warp: two block pairs
constexpr int kWarpStage = 16 * 32;            // one warp's 16 x 32 output sub-block
// the operand ring per rank: Vt | U | X per slot
template <int R>
struct Ring {
  static constexpr int VT = (kRHalf / kRBox) * (kRBox + kRPad) * R;
  static constexpr int U = 64 * (R + kRPad);
  static constexpr int X = R * (R + kXPad);
  static constexpr int SLOT = VT + U + X;
  // two slots at either rank: the producer one unit ahead. Four at rank 8 (the
  // space allows it) measured 1.5-2 % slower: operand loads further ahead of
  // their use only add traffic beside the store stream
  static constexpr int SLOTS = 2;
  static constexpr int ELEMS = SLOT * SLOTS;
};
constexpr int kMaxSlots = 4;
constexpr int kRingElems = Ring<8>::ELEMS > Ring<16>::ELEMS ? Ring<8>::ELEMS : Ring<16>::ELEMS;
constexpr size_t kRSmem = size_t(kRWarps) * kStageBufs * kWarpStage * 8 +
                          size_t(kRingElems) * 8 + size_t(2 * kMaxSlots) * 8;

struct ReconProblem {
  CUtensorMap tmVt;   // Vt items: (cols, r, items) row-major            box (132, r)
  CUtensorMap tmU;    // U rows: BLR (P, n, 1) [D_i | U_i*] panel;
                      //         batched (r, rows, items)              box (r + 4, 64)
  CUtensorMap tmOut;  // out: (cols, rows, items) row-major            box (16, 16), 128B swizzle
  const double* x;    // X_q at x + q sx, r x r row-major
  long long sx;
  int T, b;           // BLR: tiles, block (item q = off-diagonal tile in (j, i) order)
  int rank;           // the items' rank r <= R (even): rows / columns past r are zero-filled or masked
  int rblocks, halves;  // per item: 64-row blocks, 256-column halves
  int units;
  int flags;          // LRB_DEBUG_FLAGS probe bits (wrong results): 64 = skip the (UX) Vt DMMAs,
                      // 128 = no stores, 256 = no operand loads
};

// Shared-memory banking (8-byte slots, 16 per 128 B): the Vt and U fragment
// loads (row strides 132 and R + 4) put exactly two lanes on each slot, the
// minimum for 32 doubles; X rows land at stride R + 4 for the same reason; the staging stores pair each even row's lanes with the odd
// row's OTHER half of the fragment columns, so the eight lanes of a
// quarter-warp cover the eight 16-byte chunks of the swizzled line.
template <int R, bool BATCHED>
__global__ void __launch_bounds__(kRThreads, 1)
    blr_recon_kernel(const __grid_constant__ ReconProblem p) {
  constexpr int RP = R + kRPad;
  // batched: the operands may come from the previous kernel, wait for it. BLR:
  // the operands were uploaded at create and the predecessor is the diagonal
  // copy (disjoint output), so start beside it and wait only before exiting
  if (BATCHED)
    pdl_entry();
  else
    pdl_trigger();
  extern __shared__ __align__(1024) double smem[];
  // per-warp staging first (every 2 KB box 1024-B aligned for the swizzle),
  // then the operand ring (Vt | U | X per slot)
  double* stage = smem;
  double* ring = stage + size_t(kRWarps) * kStageBufs * kWarpStage;
  using L = Ring<R>;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + size_t(kRingElems));
  uint64_t* empty = full + kMaxSlots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::SLOTS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int Tm1 = p.T - 1, per_item = p.rblocks * p.halves;
  // unit -> item q, row block rb, column half; for the BLR mode also the
  // tile's block row i and its index jp among row i's off-diagonal tiles
  auto decode = [&](int u, int* q, int* i, int* jp, int* rb, int* half) {
    *q = u / per_item;
    const int w = u - *q * per_item;
    *rb = w / p.halves;
    *half = w - *rb * p.halves;
    if (BATCHED) {
      *i = *jp = 0;
    } else {
      const int j = *q / Tm1, ip = *q - j * Tm1;
      *i = ip < j ? ip : ip + 1;
      *jp = j < *i ? j : j - 1;
    }
  };

  if (warp == kRWarps) {  // the producer
    if (lane == 0) {
      const int r = p.rank;
      const uint32_t bytes =
          uint32_t((kRHalf / kRBox) * (kRBox + kRPad) * R + 64 * RP + r * r) * 8u;
      const uint64_t pol = policy_evict_normal(), pol_keep = policy_evict_last();
      int slot = 0, nq = 0;
      uint32_t phase = 0;
#pragma unroll 1
      for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++nq) {
        int q, i, jp, rb, half;
        decode(u, &q, &i, &jp, &rb, &half);
        if (nq >= L::SLOTS) mbar_wait(&empty[slot], phase ^ 1);
        double* vt = ring + size_t(slot) * L::SLOT;
        double* us = vt + L::VT;
        double* xq = us + L::U;
        if (p.flags & 256) {  // (bit 8: probe, no operand loads)
          mbar_arrive(&full[slot]);
          if (++slot == L::SLOTS) {
            slot = 0;
            phase ^= 1;
          }
          continue;
        }
        mbar_arrive_expect_tx(&full[slot], bytes);
        for (int c = 0; c < kRHalf / kRBox; ++c)
          tma_load_3d(vt + c * (kRBox + kRPad) * R, &p.tmVt, half * kRHalf + c * kRBox, 0, q,
                      &full[slot], pol_keep);
        if (BATCHED)
          tma_load_3d(us, &p.tmU, 0, rb * 64, q, &full[slot], pol);
        else
          tma_load_3d(us, &p.tmU, p.b + jp * r, i * p.b + rb * 64, 0, &full[slot], pol);
        const double* xg = p.x + q * p.sx;
        static_assert(kXPad == 0, "one contiguous copy");
        bulk_g2s(xq, xg, uint32_t(r * r * 8), &full[slot], pol);
        if (++slot == L::SLOTS) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    if (!BATCHED) pdl_wait();
    return;
  }

  const int g = lane >> 2, tq = lane & 3, odd = g & 1;
  const int rk = p.rank;
  const int row0 = (warp & 3) * 16;  // this warp's 16 rows of the 64-row block
  const int colw = (warp >> 2) * 32;  // and its 32 columns of each 64-column block
  double* wstage = stage + size_t(warp) * kStageBufs * kWarpStage;
  int slot = 0, sb = 0;  // ring slot; this warp's staging pair (0 or 1)
  uint32_t phase = 0;
#pragma unroll 1
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    int q, i, jp, rb, half;
    decode(u, &q, &i, &jp, &rb, &half);
    mbar_wait(&full[slot], phase);
    const double* vt = ring + size_t(slot) * L::SLOT;
    const double* us = vt + L::VT;
    const double* xq = us + L::U;
    // this warp's UX rows = U (16 x R) X (R x R), p ascending; the 2 * R / 8
    // chains run interleaved (both warps of a row band form the same rows: no
    // cross-warp dependency). The result stays in registers: quad shuffles
    // turn the accumulator fragments into the A fragments of the next product
    double ua[2][R / 4];
    {
      double ux[2][R / 8][2];
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int c = 0; c < R / 8; ++c) ux[f][c][0] = ux[f][c][1] = 0.0;
      // X lands r x r dense. At the template rank the reads keep their
      // compile-time pitch (a run-time pitch and mask there cost the rank-16
      // expansion 7 %); a smaller even rank reads zeros past r
      auto ux_steps = [&](auto full_rank) {
#pragma unroll
        for (int k0 = 0; k0 < R; k0 += 4) {
          double a[2], bx[R / 8];
#pragma unroll
          for (int f = 0; f < 2; ++f) a[f] = us[(row0 + 8 * f + g) * RP + k0 + tq];
#pragma unroll
          for (int c = 0; c < R / 8; ++c) {
            if constexpr (decltype(full_rank)::value)
              bx[c] = xq[(k0 + tq) * R + 8 * c + g];
            else
              bx[c] = (k0 + tq < rk && 8 * c + g < rk) ? xq[(k0 + tq) * rk + 8 * c + g] : 0.0;
          }
#pragma unroll
          for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int c = 0; c < R / 8; ++c) dmma_8x8x4(ux[f][c][0], ux[f][c][1], a[f], bx[c]);
        }
      };
      if (rk == R)
        ux_steps(std::true_type{});
      else
        ux_steps(std::false_type{});
      // A fragment (row g, column k0 + tq) = accumulator element tq % 2 of
      // lane (g, (k0 % 8) / 2 + tq / 2) in chain k0 / 8
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int kb = 0; kb < R / 4; ++kb) {
          const int src = g * 4 + ((kb & 1) << 1) + (tq >> 1);
          const double x0 = __shfl_sync(0xffffffffu, ux[f][kb >> 1][0], src);
          const double x1 = __shfl_sync(0xffffffffu, ux[f][kb >> 1][1], src);
          ua[f][kb] = (tq & 1) ? x1 : x0;
        }
    }
    // four 64 x 64 output blocks of (UX) Vt, k ascending; this warp's 16 x 32
    // part of each leaves through its own TMA stores (16 x 16 boxes).
    // Two blocks at a time: 16 independent DMMA chains per warp keep the
    // tensor pipe busy through the DMMA latency (k = R is only R / 4 deep)
#pragma unroll 1
    for (int cp = 0; cp < kRHalf / 64; cp += 2) {
      double acc[2][2][4][2];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 4; ++h) acc[e][f][h][0] = acc[e][f][h][1] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < ((p.flags & 64) ? 0 : R); k0 += 4) {
        const double a[2] = {ua[0][k0 / 4], ua[1][k0 / 4]};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cb = cp + e;
          const double* vb = vt + (cb / 2) * (kRBox + kRPad) * R + (cb % 2) * 64 + colw;
          double bv[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) bv[h] = vb[(k0 + tq) * (kRBox + kRPad) + 8 * h + g];
#pragma unroll
          for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int h = 0; h < 4; ++h)
              dmma_8x8x4(acc[e][f][h][0], acc[e][f][h][1], a[f], bv[h]);
        }
      }
      if (cp + 2 >= kRHalf / 64) {  // the slot's operands are no longer read
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
      // stage the pair (two sub-blocks) in this warp's free buffer pair: the
      // stores of the pair before the previous one have read it
      double* st = wstage + size_t(sb) * 2 * kWarpStage;
      if (lane == 0) bulk_wait_group_read<1>();
      __syncwarp();
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int box = 0; box < 2; ++box)
#pragma unroll
            for (int hs = 0; hs < 2; ++hs) {
              const int row = 8 * f + g;  // row within the warp's 16; row % 8 == g
              const int hh = hs ^ odd;    // odd rows store the other column half first
              const double v0 = odd ? acc[e][f][2 * box + (hs ^ 1)][0] : acc[e][f][2 * box + hs][0];
              const double v1 = odd ? acc[e][f][2 * box + (hs ^ 1)][1] : acc[e][f][2 * box + hs][1];
              const int chunk = (hh << 2) | tq;
              sts128(st + e * kWarpStage + box * 256 + row * 16 + ((chunk ^ g) << 1), v0, v1);
            }
      fence_proxy_async_shared_cta();
      __syncwarp();
      if (lane == 0 && !(p.flags & 128)) {  // (bit 7: probe, no stores)
        const int y0 = (BATCHED ? 0 : i * p.b) + rb * 64 + row0;
        const int z = BATCHED ? q : 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int x0 = (BATCHED ? 0 : (q / Tm1) * p.b) + half * kRHalf + (cp + e) * 64 + colw;
          tma_store_3d(&p.tmOut, st + e * kWarpStage, x0, y0, z);
          tma_store_3d(&p.tmOut, st + e * kWarpStage + 256, x0 + 16, y0, z);
        }
        bulk_commit_group();
      }
      sb ^= 1;
    }
    if (++slot == L::SLOTS) {
      slot = 0;
      phase ^= 1;
    }
  }
  if (lane == 0) bulk_wait_group0();  // the stores land before the grid completes
  if (!BATCHED) pdl_wait();  // and so does the diagonal copy before this grid
}
}  // namespace

template <bool BATCHED>
static bool launch_recon(lrb_ctx* ctx, ReconProblem& p, int64_t units, int r, cudaStream_t s,
                         lrb_status* st) {
  if (units < 1 || units > INT32_MAX) return false;
  p.units = int(units);
  p.flags = debug_flags();
  auto kern = r == 8 ? blr_recon_kernel<8, BATCHED> : blr_recon_kernel<16, BATCHED>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kRSmem));
  if (e == cudaSuccess) {
    const int64_t grid = std::min<int64_t>(ctx->sm_count, p.units);
    e = launch_pdl(kern, dim3(unsigned(grid)), dim3(kRThreads), kRSmem, s, p);
  }
  if (e != cudaSuccess) {
    *st = cuda_fail(ctx, e, "blr_recon_kernel launch");
    return true;
  }
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  *st = LRB_OK;
  return true;
}

// The whole off-diagonal part of the reconstruction in one launch, or false
// (nothing launched) when the shape is outside what the kernel serves:
// even r <= 16, b a multiple of 256, TMA-addressable buffers.
bool launch_blr_recon(lrb_ctx* ctx, const double* vtcol, const double* dcat, const double* x,
                      double* out, int64_t T, int64_t b, int64_t r, int64_t P, cudaStream_t s,
                      lrb_status* st) {
  const int64_t n = T * b, Q = T * (T - 1);
  // even ranks up to 16: the template rank R is 8 or 16, a smaller r rides on
  // the boxes' zero fill (Vt rows) and the masked X reads
  if (T < 2 || r < 2 || r > 16 || (r & 1) || b % kRHalf != 0 || Q > INT32_MAX) return false;
  const int R = r <= 8 ? 8 : 16;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  ReconProblem p;
  std::memset(&p, 0, sizeof(p));
  const bool ok = encode_c_map(&p.tmOut, out, n, n, n, 0, 1, 16) &&
                  encode_operand(&p.tmVt, vtcol, b, r, b, r * b, Q, kRBox + kRPad, R) &&
                  encode_operand(&p.tmU, dcat, P, n, P, 0, 1, R + kRPad, 64);
  if (!ok) return false;
  p.x = x;
  p.sx = r * r;
  p.T = int(T), p.b = int(b);
  p.rblocks = int(b / 64);
  p.halves = int(b / kRHalf);
  p.rank = int(r);
  return launch_recon<false>(ctx, p, Q * p.rblocks * p.halves, R, s, st);
}

// The batched expansion out_q = (U_q X_q) Vt_q (row-major items at base +
// q stride) in one launch, or false (nothing launched) outside what the kernel
// serves: even r <= 16, m a multiple of 64, n a multiple of 256, 16-byte
// aligned bases, leading dimensions and strides.
bool launch_expand_stream(lrb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t r,
                          const double* u, int64_t su, const double* x, int64_t sx,
                          const double* vt, int64_t svt, double* out, int64_t ldo, int64_t so,
                          cudaStream_t s, lrb_status* st) {
  if (r < 2 || r > 16 || (r & 1) || m % 64 != 0 || n % kRHalf != 0 || batch < 1) return false;
  const int R = r <= 8 ? 8 : 16;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0 || (batch > 1 && (sx & 1) != 0)) return false;
  const int64_t units = batch * (m / 64) * (n / kRHalf);
  if (units > INT32_MAX) return false;
  ReconProblem p;
  std::memset(&p, 0, sizeof(p));
  const bool ok = encode_c_map(&p.tmOut, out, n, m, ldo, so, batch, 16) &&
                  encode_operand(&p.tmVt, vt, n, r, n, svt, batch, kRBox + kRPad, R) &&
                  encode_operand(&p.tmU, u, r, m, r, su, batch, R + kRPad, 64);
  if (!ok) return false;
  p.x = x;
  p.sx = sx;
  p.T = 1, p.b = 0;
  p.rblocks = int(m / 64);
  p.halves = int(n / kRHalf);
  p.rank = int(r);
  return launch_recon<true>(ctx, p, units, R, s, st);
}

}  // namespace lrb
