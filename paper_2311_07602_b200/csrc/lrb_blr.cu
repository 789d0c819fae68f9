// lrb_blr.cu — block low-rank (BLR) multi-RHS matvec on the device.
//
// The reference's application caller of the batched path (proj/include/
// lrbatch/blr.hpp): a weakly admissible BLR matrix with dense diagonal tiles
// D_i (block x block) and low-rank off-diagonal tiles U_ij X_ij Vt_ij, and
//   y = M rhs    (blr_matvec :141-175, oracle blr_matvec_naive :179-202)
// with rhs, y row-major n x nrhs. Per row tile i the reference computes
//   y_i  = D_i rhs_i,   then for j != i ascending:
//   y_i += U_ij (X_ij (Vt_ij rhs_j))
// each product a naive in-order chain. On the device this is two launches of
// the batched GEMM kernels around one small coupling kernel, on one stream,
// every chain kept in the reference's order:
//   1. W_.j = [Vt_0j; Vt_1j; ...] rhs_j       strided batch over j (the tiles of
//                                            block column j stacked, one GEMM)
//   2. Z_ij = X_ij W_ij                      register-blocked r-long FMA chains
//                                            (reads W in column order, writes Z
//                                            into row i's operand block), and
//                                            rhs_i copied into the same block
//   3. y_i = [D_i | U_i0 | U_i1 | ...] [rhs_i; Z_i0; Z_i1; ...]
//      strided batch over i, K = block + (tiles-1) rank, beta 0: the
//      concatenated K runs over D's columns, then j-major then p — exactly the
//      reference's y_i = D_i rhs_i followed by its sequential per-j
//      accumulation into y_i, as ONE chain per entry.
// The device layout (stacked Vt by column, [D_i | U_i*] by row) is built once
// at lrb_blr_create.
#include <algorithm>
#include <cstring>
#include <vector>

#include "lrb_device.cuh"
#include "lrb_dispatch.cuh"
#include "lrb_internal.h"

struct lrb_blr {
  int device = 0;
  int64_t n = 0, block = 0, rank = 0, tiles = 0;
  int64_t pitch = 0;          // block + (tiles-1) rank: row pitch of d_dcat
  double* d_dcat = nullptr;   // per row i: block x pitch, [D_i | U_i0 | U_i1 | ...]
  double* d_vtcol = nullptr;  // per column j: (tiles-1) rank x block (i != j ascending)
  double* d_x = nullptr;      // same (j, i) order: rank x rank each
  // matvec workspace, grow-only (laid out for the call's nrhs inside the
  // capacity). A buffer that is outgrown is retired, not freed: a captured
  // graph may still reference it; retired buffers and plans are released by
  // lrb_blr_destroy. ws_ev orders the matrix's eager matvecs on different
  // streams (they share d_w / d_rz).
  size_t w_cap = 0, rz_cap = 0;  // doubles
  // odd right-hand-side counts: rhs / y copies with one more (zero) column,
  // so the fused matvec's 16-byte operand rule holds
  double* d_rpad = nullptr;
  double* d_ypad = nullptr;
  size_t rpad_cap = 0, ypad_cap = 0;
  double* d_w = nullptr;
  double* d_rz = nullptr;     // per row i: pitch x nrhs, [rhs_i; Z_i0; Z_i1; ...]
  cudaEvent_t ws_ev = nullptr;
  bool ws_pending = false;
  // the fused matvec's sync words: [T][4] ready counts (row i, quarter of its
  // Z columns; they only ever grow, a launch waits for epoch + 1 times the
  // quarter's size), then three 64-bit words: tickets, finished CTAs (both
  // reset by the last CTA out) and the epoch (allocated and zeroed at create)
  unsigned* d_sync = nullptr;
  std::vector<void*> retired;
  std::vector<lrb_ptr_plan*> retired_plans;
  // reconstruct_dense: UX tiles in Vt's (j, i) order and the tile plan for
  // the last output buffer
  double* d_ux = nullptr;
  const double* recon_out = nullptr;
  lrb_ptr_plan* recon_plan = nullptr;
};

namespace lrb {
bool launch_blr_fused(lrb_ctx* ctx, const double* rhs, int64_t nrhs, int64_t ld, double* y,
                      int64_t T,
                      int64_t b, int64_t r, int64_t P, const double* vtcol, const double* x,
                      const double* dcat, double* rz, unsigned* ready,
                      unsigned long long* next, cudaStream_t s, lrb_status* st);
bool blr_fused_shape_ok(int64_t T, int64_t b, int64_t r, int64_t nrhs);
bool launch_blr_recon(lrb_ctx* ctx, const double* vtcol, const double* dcat, const double* x,
                      double* out, int64_t T, int64_t b, int64_t r, int64_t P, cudaStream_t s,
                      lrb_status* st);
lrb_status run_strided_rowmajor_beta(lrb_ctx* ctx, int64_t m, int64_t n, int64_t k,
                                     const double* A, int64_t lda, int64_t sA, const double* B,
                                     int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC,
                                     int64_t batch, int beta_one, cudaStream_t stream);
}

using lrb::fail;

namespace {

// everything the matrix owns, after the device is idle (lrb_blr_destroy)
void free_all(lrb_ctx* ctx, lrb_blr* m) {
  cudaDeviceSynchronize();
  if (m->recon_plan) lrb_ptr_plan_destroy(ctx, m->recon_plan);
  for (lrb_ptr_plan* p : m->retired_plans) lrb_ptr_plan_destroy(ctx, p);
  for (void* p : m->retired) cudaFree(p);
  if (m->d_ux) cudaFree(m->d_ux);
  if (m->d_w) cudaFree(m->d_w);
  if (m->d_rz) cudaFree(m->d_rz);
  if (m->d_rpad) cudaFree(m->d_rpad);
  if (m->d_ypad) cudaFree(m->d_ypad);
  if (m->ws_ev) cudaEventDestroy(m->ws_ev);
  if (m->d_sync) cudaFree(m->d_sync);
  m->d_sync = nullptr;
  m->retired.clear();
  m->retired_plans.clear();
  m->recon_plan = nullptr;
  m->d_ux = m->d_w = m->d_rz = m->d_rpad = m->d_ypad = nullptr;
  m->ws_ev = nullptr;
}

// grow-only: a capacity that is outgrown retires the old buffer
lrb_status grow(lrb_ctx* ctx, lrb_blr* m, double** buf, size_t* cap, size_t need) {
  if (*cap >= need && *buf) return LRB_OK;
  if (*buf) m->retired.push_back(*buf);
  *buf = nullptr;
  *cap = 0;
  // a plain allocation even while a graph is being captured on this thread
  // (relaxed mode): the graph then references it like any caller buffer
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  cudaError_t e = cudaMalloc(buf, need * sizeof(double));
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return lrb::cuda_fail(ctx, e, "lrb_blr workspace");
  *cap = need;
  return LRB_OK;
}

lrb_status ensure_ws(lrb_ctx* ctx, lrb_blr* m, int64_t nrhs) {
  const int64_t T = m->tiles, r = m->rank, items = T * (T - 1);
  lrb_status st = grow(ctx, m, &m->d_w, &m->w_cap, size_t(std::max<int64_t>(1, items * r * nrhs)));
  if (st) return st;
  return grow(ctx, m, &m->d_rz, &m->rz_cap, size_t(T * m->pitch * nrhs));
}

// Step 3: Z_ij = X_ij W_ij for every off-diagonal tile. Item q runs in W's
// (column j, row i != j) order; its Z block goes to row i's slot jp. Each
// thread owns one entry Z[p][c] = sum_k X[p][k] W[k][c] as an in-order FMA
// chain from zero (the order DMMA and the FMA-chain oracle use). Bytes: X
// r^2 + W r*nrhs read, Z r*nrhs written per item — a few MB in total.
// Warp-per-item form for small items (r^2 + r*nrhs <= kCoupleSmem doubles):
// the warp stages X_q and W_q in shared memory with all its loads in flight,
// then computes Z_q as the same r-long chains (k ascending, from 0): on DMMA
// 8x8x4 tiles when r and nrhs are multiples of 8, else one entry per lane.
// The register-blocked kernel below (scalar chains straight from global
// memory) and a scalar shared-memory form both measured 16-18 us per matvec
// on the 16-RHS bench shape, bound by one load per FMA.
constexpr int kCoupleSmem = 512;  // doubles per warp (8 warps: 32 KB static)
template <bool MMA>
__global__ void __launch_bounds__(256) blr_couple_warp_kernel(const double* __restrict__ x,
                                                              const double* __restrict__ w,
                                                              const double* __restrict__ rhs,
                                                              double* __restrict__ rz, int tiles,
                                                              int block, int rank, int nrhs) {
  lrb::pdl_entry_ordered();  // the row step reads rhs before its own wait
  __shared__ double sm[8][kCoupleSmem];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Q = tiles * (tiles - 1);
  const int rr = rank * rank, per = rank * nrhs;
  const int64_t pitch = block + int64_t(tiles - 1) * rank;
  // rhs_i into the first block rows of row i's operand block (contiguous
  // b * nrhs doubles both sides), spread over the whole grid, four
  // independent loads per thread in flight; skipped (rhs null) when the row
  // step reads rhs directly (BlrRowProblem)
  if (rhs) {
    const int64_t tile_elems = int64_t(block) * nrhs, total = int64_t(tiles) * tile_elems;
    const int64_t step = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e0 < total; e0 += 4 * step) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * step;
        v[u] = e < total ? __ldg(rhs + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * step;
        if (e < total) {
          const int64_t i = e / tile_elems;
          rz[e + i * (pitch - block) * nrhs] = v[u];
        }
      }
    }
  }
  double* xs = sm[warp];
  double* ws = xs + rr;
  for (int q = blockIdx.x * 8 + warp; q < Q; q += gridDim.x * 8) {
    const double* xq = x + int64_t(q) * rr;
    const double* wq = w + int64_t(q) * per;
    // all of the item's loads in flight at once (a rolled loop would wait
    // one DRAM round trip per 32 elements)
    double v[kCoupleSmem / 32];
#pragma unroll
    for (int t = 0; t < kCoupleSmem / 32; ++t) {
      const int e = lane + 32 * t;
      v[t] = e < rr ? __ldg(xq + e) : (e - rr < per ? __ldg(wq + (e - rr)) : 0.0);
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kCoupleSmem / 32; ++t) {
      const int e = lane + 32 * t;
      if (e < rr + per) xs[e] = v[t];  // ws == xs + rr
    }
    __syncwarp();
    const int j = q / (tiles - 1), ip = q - j * (tiles - 1);
    const int i = ip < j ? ip : ip + 1;
    const int jp = j < i ? j : j - 1;
    double* zq = rz + (int64_t(i) * pitch + block + int64_t(jp) * rank) * nrhs;
    if (MMA) {
      // r and nrhs multiples of 8: each 8 x 8 tile of Z is a chain of r/4
      // DMMA 8x8x4 steps in ascending k (an in-order FMA chain per entry,
      // bitwise the scalar form); lane (g, t) holds Z[p0+g][c0+2t .. +1]
      const int g = lane >> 2, t = lane & 3;
      for (int p0 = 0; p0 < rank; p0 += 8)
        for (int c0 = 0; c0 < nrhs; c0 += 8) {
          double d0 = 0.0, d1 = 0.0;
          for (int k0 = 0; k0 < rank; k0 += 4)
            lrb::dmma_8x8x4(d0, d1, xs[(p0 + g) * rank + k0 + t], ws[(k0 + t) * nrhs + c0 + g]);
          *reinterpret_cast<double2*>(zq + (p0 + g) * nrhs + c0 + 2 * t) = make_double2(d0, d1);
        }
    } else {
      for (int e = lane; e < per; e += 32) {
        const int p = e / nrhs, c = e - p * nrhs;
        double acc = 0.0;
        for (int k = 0; k < rank; ++k) acc = fma(xs[p * rank + k], ws[k * nrhs + c], acc);
        zq[e] = acc;
      }
    }
  }
}

template <int CP>
__global__ void __launch_bounds__(256) blr_couple_kernel(const double* __restrict__ x,
                                                         const double* __restrict__ w,
                                                         const double* __restrict__ rhs,
                                                         double* __restrict__ rz, int tiles,
                                                         int block, int rank, int nrhs) {
  lrb::pdl_entry_ordered();  // the row step reads rhs before its own wait
  // a thread owns a 4-row x CP-column block of one Z_q (CP = 2 when nrhs is
  // even): per step k it loads four X values and one W pair for 4*CP FMAs;
  // every entry is still one r-long chain over k ascending. 32-bit indices:
  // Q = tiles*(tiles-1) items of r*nrhs entries.
  constexpr int RP = 4;
  const int rg_n = (rank + RP - 1) / RP, cg_n = nrhs / CP;
  const int per_item = rg_n * cg_n, per = rank * nrhs;
  const int Q = tiles * (tiles - 1);
  const int total = Q * per_item;
  const int64_t pitch = block + int64_t(tiles - 1) * rank;
  // rhs_i into the first block rows of row i's operand block
  const int64_t n_rhs = int64_t(tiles) * block * nrhs;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; rhs && e < n_rhs;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / (int64_t(block) * nrhs), rem = e - i * block * nrhs;
    rz[i * pitch * nrhs + rem] = __ldg(rhs + e);
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int q = t / per_item, rem = t - q * per_item;
    const int rg = rem / cg_n, cg = rem - rg * cg_n;
    const int p0 = rg * RP, c0 = cg * CP;
    const int j = q / (tiles - 1), ip = q - j * (tiles - 1);
    const int i = ip < j ? ip : ip + 1;
    const int jp = j < i ? j : j - 1;
    const double* xq = x + int64_t(q) * rank * rank;
    const double* wq = w + int64_t(q) * per + c0;
    const double* xr[RP];
#pragma unroll
    for (int a = 0; a < RP; ++a) xr[a] = xq + min(p0 + a, rank - 1) * rank;
    double acc[RP][CP];
#pragma unroll
    for (int a = 0; a < RP; ++a)
#pragma unroll
      for (int c = 0; c < CP; ++c) acc[a][c] = 0.0;
#pragma unroll 2
    for (int k = 0; k < rank; ++k) {
      double wv[CP];
      if constexpr (CP == 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(wq + k * nrhs));
        wv[0] = v.x;
        wv[1] = v.y;
      } else {
        wv[0] = __ldg(wq + k * nrhs);
      }
#pragma unroll
      for (int a = 0; a < RP; ++a) {
        const double xv = __ldg(xr[a] + k);
#pragma unroll
        for (int c = 0; c < CP; ++c) acc[a][c] = fma(xv, wv[c], acc[a][c]);
      }
    }
    double* zq = rz + (int64_t(i) * pitch + block + int64_t(jp) * rank) * nrhs + c0;
#pragma unroll
    for (int a = 0; a < RP; ++a)
      if (p0 + a < rank) {
#pragma unroll
        for (int c = 0; c < CP; ++c) zq[(p0 + a) * nrhs + c] = acc[a][c];
      }
  }
}

// reconstruct_dense step 1: UX_p = U_ij X_ij for every off-diagonal tile, p
// in Vt's (column j, row i != j) order, U_ij read from the concatenated row
// layout [D_i | U_i0 | U_i1 | ...]. One block per item (32-bit indices within it).
// A thread owns a 4-row x CP-column block of UX (CP = 2 when rank is even):
// per step q it loads four U values and one X pair for 4*CP FMAs. Every
// entry is still one r-long FMA chain over q ascending.
template <int CP>
__global__ void __launch_bounds__(256) blr_ux_kernel(const double* __restrict__ dcat,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ ux, int tiles,
                                                     int block, int rank) {
  lrb::pdl_entry();
  constexpr int RP = 4;
  const int Q = tiles * (tiles - 1);
  const int64_t K = block + int64_t(tiles - 1) * rank;  // row pitch of [D_i | U_i*]
  const int row_groups = (block + RP - 1) / RP, col_groups = rank / CP;
  const int work = row_groups * col_groups;
  for (int p = blockIdx.x; p < Q; p += gridDim.x) {
    const int j = p / (tiles - 1), ip = p - j * (tiles - 1);
    const int i = ip < j ? ip : ip + 1;
    const int jp = j < i ? j : j - 1;
    const double* ub = dcat + int64_t(i) * block * K + block + int64_t(jp) * rank;
    const double* xb = x + int64_t(p) * rank * rank;
    double* out = ux + int64_t(p) * block * rank;
    for (int wkr = threadIdx.x; wkr < work; wkr += blockDim.x) {
      const int rg = wkr / col_groups, cg = wkr - rg * col_groups;
      const int r0 = rg * RP, c0 = cg * CP;
      double acc[RP][CP];
#pragma unroll
      for (int a = 0; a < RP; ++a)
#pragma unroll
        for (int c = 0; c < CP; ++c) acc[a][c] = 0.0;
      const double* ur[RP];
#pragma unroll
      for (int a = 0; a < RP; ++a) ur[a] = ub + int64_t(min(r0 + a, block - 1)) * K;
#pragma unroll 2
      for (int q = 0; q < rank; ++q) {
        double xv[CP];
        if constexpr (CP == 2) {
          const double2 t = __ldg(reinterpret_cast<const double2*>(xb + q * rank + c0));
          xv[0] = t.x;
          xv[1] = t.y;
        } else {
          xv[0] = __ldg(xb + q * rank + c0);
        }
#pragma unroll
        for (int a = 0; a < RP; ++a) {
          const double u = __ldg(ur[a] + q);
#pragma unroll
          for (int c = 0; c < CP; ++c) acc[a][c] = fma(u, xv[c], acc[a][c]);
        }
      }
#pragma unroll
      for (int a = 0; a < RP; ++a)
        if (r0 + a < block) {
#pragma unroll
          for (int c = 0; c < CP; ++c) out[(r0 + a) * rank + c0 + c] = acc[a][c];
        }
    }
  }
}

// reconstruct_dense step 1 on DMMA (r % 8 == 0, b % 8 == 0, r <= 32): one
// block per item; X_ij staged in shared memory; warp w takes 8-row groups of
// UX and runs each 8 x 8 tile as r/4 DMMA 8x8x4 steps in ascending q (the
// same in-order chains as the scalar kernel above, which measured 66 us on
// the 16384 / 512 / 16 reconstruction at 1.3 TB/s). Each U value is loaded
// once per item, straight from the [D_i | U_i*] row panel.
__global__ void __launch_bounds__(256) blr_ux_mma_kernel(const double* __restrict__ dcat,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ ux, int tiles,
                                                         int block, int rank) {
  lrb::pdl_entry();
  __shared__ double xs[32 * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int Q = tiles * (tiles - 1);
  const int64_t K = block + int64_t(tiles - 1) * rank;  // row pitch of [D_i | U_i*]
  const int ct_n = rank / 8;
  for (int p = blockIdx.x; p < Q; p += gridDim.x) {
    const int j = p / (tiles - 1), ip = p - j * (tiles - 1);
    const int i = ip < j ? ip : ip + 1;
    const int jp = j < i ? j : j - 1;
    const double* ub = dcat + int64_t(i) * block * K + block + int64_t(jp) * rank;
    double* out = ux + int64_t(p) * block * rank;
    __syncthreads();  // the previous item's X is no longer read
    for (int e = threadIdx.x; e < rank * rank; e += blockDim.x)
      xs[e] = __ldg(x + int64_t(p) * rank * rank + e);
    __syncthreads();
    for (int p0 = warp * 8; p0 < block; p0 += 64) {
      double d[4][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = 0.0;
      const double* urow = ub + int64_t(p0 + g) * K + t;
      for (int k0 = 0; k0 < rank; k0 += 4) {
        const double a = __ldg(urow + k0);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < ct_n) lrb::dmma_8x8x4(d[c][0], d[c][1], a, xs[(k0 + t) * rank + 8 * c + g]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < ct_n)
          *reinterpret_cast<double2*>(out + (p0 + g) * rank + 8 * c + 2 * t) =
              make_double2(d[c][0], d[c][1]);
    }
  }
}

// reconstruct_dense: the diagonal tiles into the n x n row-major output, one
// warp per tile row, 16-byte accesses when the rows allow them. One CTA per SM
// leaves room for the streaming off-diagonal kernel, which starts beside it
// (it waits for this grid only before it exits: disjoint outputs), so the
// copy's bandwidth overlaps that kernel's DMMA work. The copy waits for its
// own predecessor before it lets the streaming kernel launch (write-after-
// read on `out`).
__global__ void __launch_bounds__(256) blr_diag_kernel(const double* __restrict__ dcat,
                                                       double* __restrict__ out, int tiles,
                                                       int block, int64_t pitch, int vec) {
  lrb::pdl_entry_ordered();
  const int64_t n = int64_t(tiles) * block;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int g = blockIdx.x * wpb + warp; g < tiles * block; g += gridDim.x * wpb) {
    const int t = g / block, row = g - t * block;
    const double* src = dcat + int64_t(g) * pitch;
    double* dst = out + (int64_t(t) * block + row) * n + int64_t(t) * block;
    if (vec) {
#pragma unroll 4
      for (int c = 2 * lane; c < block; c += 64)
        *reinterpret_cast<double2*>(dst + c) = __ldg(reinterpret_cast<const double2*>(src + c));
    } else {
      for (int c = lane; c < block; c += 32) dst[c] = __ldg(src + c);
    }
  }
}

}  // namespace

extern "C" lrb_status lrb_blr_create(lrb_ctx* ctx, int64_t n, int64_t block, int64_t rank,
                                     const double* diag, const double* u, const double* x,
                                     const double* vt, lrb_blr** out) {
  static const char* fn = "lrb_blr_create";
  if (!out) return fail(ctx, LRB_ERR_ARG, "%s: out is null", fn);
  *out = nullptr;
  // BlrMatrix constructor invariants (blr.hpp:23-31), with its messages
  if (!(block >= 1 && n >= block)) return fail(ctx, LRB_ERR_SHAPE, "BlrMatrix: bad block size");
  if (n % block != 0)
    return fail(ctx, LRB_ERR_SHAPE, "BlrMatrix: n = %lld is not a multiple of block_size %lld",
                (long long)n, (long long)block);
  if (!(rank >= 1 && rank <= block))
    return fail(ctx, LRB_ERR_SHAPE, "BlrMatrix: rank must be in [1, block]");
  const int64_t T = n / block;
  if (n >= (int64_t(1) << 31))
    return fail(ctx, LRB_ERR_UNSUPPORTED, "%s: n = %lld exceeds 2^31 - 1", fn, (long long)n);
  if (!diag || (T > 1 && (!u || !x || !vt)))
    return fail(ctx, LRB_ERR_ARG, "%s: a tile array is null", fn);
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "%s: null ctx", fn);
  lrb_status st = lrb::bind(ctx);
  if (st) return st;
  auto* m = new (std::nothrow) lrb_blr;
  if (!m) return fail(ctx, LRB_ERR_CAPACITY, "%s: out of host memory", fn);
  m->device = ctx->device;
  m->n = n;
  m->block = block;
  m->rank = rank;
  m->tiles = T;
  const int64_t b = block, r = rank, items = T * (T - 1);
  auto upload = [&](double** dst, const std::vector<double>& h) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, h.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(*dst, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
    return e;
  };
  const int64_t P = b + (T - 1) * r;  // [D_i | U_i0 | U_i1 | ...] row pitch
  m->pitch = P;
  // reference off-diagonal order: row-major over (i, j != i) (blr.hpp:33-35)
  auto off = [&](int64_t i, int64_t j) { return i * (T - 1) + (j < i ? j : j - 1); };
  std::vector<double> dcat(size_t(T * b * P));
  for (int64_t i = 0; i < T; ++i)
    for (int64_t row = 0; row < b; ++row) {
      std::memcpy(&dcat[size_t((i * b + row) * P)], diag + (i * b + row) * b,
                  size_t(b) * sizeof(double));
      for (int64_t j = 0; j < T; ++j) {
        if (i == j) continue;
        const int64_t jp = j < i ? j : j - 1;
        const double* uij = u + off(i, j) * b * r;  // block x rank, row-major
        std::memcpy(&dcat[size_t((i * b + row) * P + b + jp * r)], uij + row * r,
                    size_t(r) * sizeof(double));
      }
    }
  cudaError_t e = upload(&m->d_dcat, dcat);
  if (e == cudaSuccess && T > 1) {
    const size_t sync_bytes = size_t(T) * 16 + 32;
    e = cudaMalloc(&m->d_sync, sync_bytes);
    if (e == cudaSuccess) e = cudaMemset(m->d_sync, 0, sync_bytes);
  }
  if (e == cudaSuccess && T > 1) {
    std::vector<double> vtcol(size_t(items * r * b)), xs(size_t(items * r * r));
    int64_t q = 0;
    for (int64_t j = 0; j < T; ++j)
      for (int64_t i = 0; i < T; ++i) {
        if (i == j) continue;
        const int64_t o = off(i, j);
        std::memcpy(&vtcol[size_t(q * r * b)], vt + o * r * b, size_t(r * b) * sizeof(double));
        std::memcpy(&xs[size_t(q * r * r)], x + o * r * r, size_t(r * r) * sizeof(double));
        ++q;
      }
    e = upload(&m->d_vtcol, vtcol);
    if (e == cudaSuccess) e = upload(&m->d_x, xs);
  }
  if (e != cudaSuccess) {
    lrb_blr_destroy(ctx, m);
    return lrb::cuda_fail(ctx, e, "lrb_blr_create: upload");
  }
  *out = m;
  return LRB_OK;
}

namespace {
lrb_status matvec_steps(lrb_ctx* ctx, lrb_blr* m, const double* rhs, int64_t nrhs, double* y,
                        cudaStream_t s);
}

extern "C" lrb_status lrb_blr_matvec_device(lrb_ctx* ctx, lrb_blr* m, const double* rhs,
                                            int64_t nrhs, double* y, void* stream) {
  static const char* fn = "lrb_blr_matvec";
  if (!ctx || !m) return fail(ctx, LRB_ERR_ARG, "%s: null ctx or matrix", fn);
  if (nrhs < 1) return fail(ctx, LRB_ERR_SHAPE, "%s: nrhs must be >= 1", fn);
  if (!rhs || !y) return fail(ctx, LRB_ERR_ARG, "%s: rhs or y is null", fn);
  lrb_status st = lrb::bind(ctx);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t T = m->tiles, b = m->block, P = m->pitch;
  if (T == 1)  // y = D rhs only
    return lrb::run_strided_rowmajor_beta(ctx, b, nrhs, b, m->d_dcat, P, b * P, rhs, nrhs,
                                          b * nrhs, y, nrhs, b * nrhs, T, 0, s);
  st = ensure_ws(ctx, m, nrhs);
  if (st) return st;
  // eager calls on different streams share the workspace: wait for the last
  // user (captured calls are ordered by the graph's own stream)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  LRB_CUDA_TRY(ctx, cudaStreamIsCapturing(s, &cap));
  const bool eager = cap == cudaStreamCaptureStatusNone;
  if (eager && m->ws_pending) LRB_CUDA_TRY(ctx, cudaStreamWaitEvent(s, m->ws_ev, 0));
  st = matvec_steps(ctx, m, rhs, nrhs, y, s);
  if (st) return st;
  if (eager) {
    if (!m->ws_ev) LRB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&m->ws_ev, cudaEventDisableTiming));
    LRB_CUDA_TRY(ctx, cudaEventRecord(m->ws_ev, s));
    m->ws_pending = true;
  }
  return LRB_OK;
}

namespace {
// dst (rows x kd, row-major) = the first min(ks, kd) columns of src (rows x
// ks), further columns zero: the odd-count matvec's padded copies
__global__ void __launch_bounds__(256) blr_repitch_kernel(const double* __restrict__ src, int ks,
                                                          double* __restrict__ dst, int kd,
                                                          int64_t rows) {
  lrb::pdl_entry();
  const int64_t total = rows * kd;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = e / kd;
    const int c = int(e - row * kd);
    dst[e] = c < ks ? src[row * ks + c] : 0.0;
  }
}

lrb_status matvec_steps(lrb_ctx* ctx, lrb_blr* m, const double* rhs, int64_t nrhs, double* y,
                        cudaStream_t s) {
  lrb_status st = LRB_OK;
  const int64_t T = m->tiles, b = m->block, r = m->rank, K = (T - 1) * r, P = m->pitch;
  // An odd count (the plain matvec, nrhs = 1, first of all) leaves rhs and y
  // rows that are not 16-byte multiples, which TMA cannot address: every
  // launch form would fall to its per-lane loaders (0.3 of HBM). Run the even
  // count on copies with one more, zero, column instead. Every column's
  // chains are its own, so the results are the unpadded ones bit for bit,
  // and the two copies move n x nrhs doubles against the whole matrix.
  if (nrhs & 1) {
    const int64_t n = T * b, k2 = nrhs + 1;
    st = ensure_ws(ctx, m, k2);
    if (!st) st = grow(ctx, m, &m->d_rpad, &m->rpad_cap, size_t(n * k2));
    if (!st) st = grow(ctx, m, &m->d_ypad, &m->ypad_cap, size_t(n * k2));
    if (st) return st;
    const unsigned blocks = unsigned(std::min<int64_t>((n * k2 + 255) / 256, 148 * 8));
    LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_repitch_kernel, dim3(blocks), dim3(256), 0, s, rhs,
                                      int(nrhs), m->d_rpad, int(k2), n));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
    st = matvec_steps(ctx, m, m->d_rpad, k2, m->d_ypad, s);
    if (st) return st;
    LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_repitch_kernel, dim3(blocks), dim3(256), 0, s,
                                      static_cast<const double*>(m->d_ypad), int(k2), y,
                                      int(nrhs), n));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
    return LRB_OK;
  }
  // one persistent launch when the shape allows it (lrb_blr_fused.cu);
  // LRB_BLR_FUSED=0 or debug bit 9 keeps the three-launch form below
  const char* fe = std::getenv("LRB_BLR_FUSED");
  if (!(fe && fe[0] == '0') && !(lrb::debug_flags() & 512) && m->d_sync) {
    unsigned* ready = m->d_sync;
    auto* next = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(m->d_sync) + size_t(T) * 16);
    if (lrb::launch_blr_fused(ctx, rhs, nrhs, nrhs, y, T, b, r, P, m->d_vtcol, m->d_x, m->d_dcat,
                              m->d_rz, ready, next, s, &st))
      return st;
    // More than 16 right-hand sides: the same launch over column ranges of 16
    // (the last one shorter), the matrix streamed once per range. Measured
    // against the three launches' wide-tile forms at 18..64 columns: 27-30 %
    // faster at rank 16 and 32 (n16384 b256 r16 k32 0.155 -> 0.112 ms, b512
    // r16 0.115 -> 0.080, b512 r32 0.167 -> 0.124), 11 % slower at rank 8
    // (n32768 b512 r8 k32 0.130 vs 0.146), hence the rank gate.
    if (nrhs > 16 && nrhs <= 64 && r >= 16 && lrb::blr_fused_shape_ok(T, b, r, 16)) {
      bool all = true;
      for (int64_t c0 = 0; c0 < nrhs && all; c0 += 16) {
        const int64_t w = std::min<int64_t>(16, nrhs - c0);
        all = lrb::launch_blr_fused(ctx, rhs + c0, w, nrhs, y + c0, T, b, r, P, m->d_vtcol, m->d_x,
                                    m->d_dcat, m->d_rz, ready, next, s, &st);
        if (all && st) return st;
        if (!all && c0 > 0)  // (cannot happen: every range has the first one's alignment)
          return fail(ctx, LRB_ERR_UNSUPPORTED, "lrb_blr_matvec: column range %lld not addressable",
                      (long long)c0);
      }
      if (all) return LRB_OK;
    }
  }
  // 1. W_.j = [Vt_ij]_i rhs_j
  st = lrb::run_strided_rowmajor_beta(ctx, K, nrhs, b, m->d_vtcol, b, K * b, rhs, nrhs, b * nrhs,
                                      m->d_w, nrhs, K * nrhs, T, 0, s);
  if (st) return st;
  // 3 (prepared first): the row step as a BlrRowProblem when its operands
  // are TMA-addressable and b is a multiple of the 64-deep chunks: it reads
  // rhs itself and starts its D_i rhs_i part while step 2 still runs
  lrb::BlrRowProblem rp;
  std::memset(&rp, 0, sizeof(rp));
  using RowCfg8 = lrb::VariantTraits<LRB_V_M8K64>::Cfg<false, false, true>;
  using RowCfg16 = lrb::VariantTraits<LRB_V_M16K64>::Cfg<false, false, true>;
  const int mb = nrhs <= 8 ? RowCfg8::MB : RowCfg16::MB;
  const bool row_ok =
      nrhs <= 16 && b % RowCfg16::KB == 0 && !(lrb::debug_flags() & 256) &&
      lrb::encode_operand(&rp.tmA, rhs, nrhs, b, nrhs, b * nrhs, T, mb + lrb::kPad,
                          RowCfg16::KB) &&
      lrb::encode_operand(&rp.tmA2, m->d_rz + b * nrhs, nrhs, K, nrhs, P * nrhs, T,
                          mb + lrb::kPad, RowCfg16::KB) &&
      lrb::encode_operand(&rp.tmB, m->d_dcat, P, b, P, b * P, T, RowCfg16::KB + lrb::kPad,
                          RowCfg16::NB);
  const double* copy_src = row_ok ? nullptr : rhs;
  // 2. Z_ij = X_ij W_ij into [rhs_i; Z_i*] (and rhs_i copied there for the
  //    strided fallback of step 3)
  if (r * r + r * nrhs <= kCoupleSmem) {
    const int64_t blocks = std::min<int64_t>((T * (T - 1) + 7) / 8, int64_t(ctx->sm_count) * 8);
    // Z rows land 16-byte aligned when b and r are even (pitch, offsets)
    if (r % 8 == 0 && nrhs % 8 == 0)
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_couple_warp_kernel<true>, dim3(unsigned(blocks)),
                                        dim3(256), 0, s, m->d_x, m->d_w, copy_src, m->d_rz,
                                        int(T), int(b), int(r), int(nrhs)));
    else
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_couple_warp_kernel<false>, dim3(unsigned(blocks)),
                                        dim3(256), 0, s, m->d_x, m->d_w, copy_src, m->d_rz,
                                        int(T), int(b), int(r), int(nrhs)));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
  } else {
    const int cp = (nrhs % 2 == 0) ? 2 : 1;
    const int64_t work = std::max(T * (T - 1) * ((r + 3) / 4) * (nrhs / cp), T * b * nrhs);
    const int64_t blocks = std::min<int64_t>((work + 255) / 256, int64_t(ctx->sm_count) * 16);
    if (cp == 2)
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_couple_kernel<2>, dim3(unsigned(blocks)), dim3(256), 0,
                                        s, m->d_x, m->d_w, copy_src, m->d_rz, int(T), int(b),
                                        int(r), int(nrhs)));
    else
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_couple_kernel<1>, dim3(unsigned(blocks)), dim3(256), 0,
                                        s, m->d_x, m->d_w, copy_src, m->d_rz, int(T), int(b),
                                        int(r), int(nrhs)));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
  }
  // 3. y_i = [D_i | U_i*] [rhs_i; Z_i*]: one chain per entry over D's columns,
  //    then the off-diagonal blocks j-major
  if (row_ok) {
    rp.C = y;
    rp.m = int(nrhs);
    rp.n = int(b);
    rp.k = int(P);
    rp.kb = int(b);
    rp.tiles_i = 1;
    rp.tiles_per_item = int((b + RowCfg16::NB - 1) / RowCfg16::NB);
    rp.num_tiles = T * rp.tiles_per_item;
    lrb::LaunchInfo info{0, 0};
    if (nrhs <= 8)
      LRB_CUDA_TRY(ctx, lrb::launch_gemm<RowCfg8>(rp, 0, ctx->device, ctx->sm_count, s, &info));
    else
      LRB_CUDA_TRY(ctx, lrb::launch_gemm<RowCfg16>(rp, 0, ctx->device, ctx->sm_count, s, &info));
    if (info.grid > 0) ctx->launches.fetch_add(1, std::memory_order_relaxed);
    return LRB_OK;
  }
  return lrb::run_strided_rowmajor_beta(ctx, b, nrhs, P, m->d_dcat, P, b * P, m->d_rz, nrhs,
                                        P * nrhs, y, nrhs, b * nrhs, T, 0, s);
}
}  // namespace

extern "C" lrb_status lrb_blr_matvec(lrb_ctx* ctx, lrb_blr* m, const double* rhs, int64_t nrhs,
                                     double* y) {
  if (!ctx || !m) return fail(ctx, LRB_ERR_ARG, "lrb_blr_matvec: null ctx or matrix");
  if (nrhs < 1) return fail(ctx, LRB_ERR_SHAPE, "lrb_blr_matvec: nrhs must be >= 1");
  if (!rhs || !y) return fail(ctx, LRB_ERR_ARG, "lrb_blr_matvec: rhs or y is null");
  lrb_status st = lrb::bind(ctx);
  if (st) return st;
  const size_t bytes = size_t(m->n * nrhs) * sizeof(double);
  double *d_rhs = nullptr, *d_y = nullptr;
  cudaStream_t s = ctx->lane_stream[0];
  LRB_CUDA_TRY(ctx, lrb::pool_alloc(ctx, reinterpret_cast<void**>(&d_rhs), bytes, s));
  LRB_CUDA_TRY(ctx, lrb::pool_alloc(ctx, reinterpret_cast<void**>(&d_y), bytes, s));
  cudaError_t e = cudaMemcpyAsync(d_rhs, rhs, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    st = lrb_blr_matvec_device(ctx, m, d_rhs, nrhs, d_y, s);
    if (!st) e = cudaMemcpyAsync(y, d_y, bytes, cudaMemcpyDeviceToHost, s);
  }
  cudaFreeAsync(d_rhs, s);
  cudaFreeAsync(d_y, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (st) return st;
  if (e != cudaSuccess) return lrb::cuda_fail(ctx, e, "lrb_blr_matvec: copy");
  if (e2 != cudaSuccess) return lrb::cuda_fail(ctx, e2, "lrb_blr_matvec: sync");
  return LRB_OK;
}

extern "C" lrb_status lrb_blr_destroy(lrb_ctx* ctx, lrb_blr* m) {
  if (!m) return LRB_OK;
  if (ctx) cudaSetDevice(ctx->device);
  free_all(ctx, m);
  if (m->d_dcat) cudaFree(m->d_dcat);
  if (m->d_vtcol) cudaFree(m->d_vtcol);
  if (m->d_x) cudaFree(m->d_x);
  delete m;
  return LRB_OK;
}

// BlrMatrix::reconstruct_dense (blr.hpp:62-86) on the device: diagonal tiles
// copied; off-diagonal tiles (U X) Vt in the reference's order — UX by
// blr_ux_kernel, then the b x b tiles by one launch of the batched GEMM kernel
// (q64 tiles, K = rank) over a BlrTileProblem that writes straight into the
// n x n output, through the TMA-store epilogue when rank <= 16 (the
// write-bound case) and the output is TMA-aligned. Operands that TMA cannot
// address (odd rank or block) take a pointer-array plan instead.
extern "C" lrb_status lrb_blr_reconstruct_dense(lrb_ctx* ctx, lrb_blr* m, double* out,
                                                int on_device, void* stream) {
  static const char* fn = "lrb_blr_reconstruct_dense";
  if (!ctx || !m) return fail(ctx, LRB_ERR_ARG, "%s: null ctx or matrix", fn);
  if (!out) return fail(ctx, LRB_ERR_ARG, "%s: out is null", fn);
  lrb_status st = lrb::bind(ctx);
  if (st) return st;
  const int64_t T = m->tiles, b = m->block, r = m->rank, n = m->n;
  if (!on_device) {
    // host destination: through a pooled device buffer, synchronously
    cudaStream_t s = ctx->lane_stream[0];
    double* d = nullptr;
    const size_t bytes = size_t(n) * size_t(n) * sizeof(double);
    LRB_CUDA_TRY(ctx, lrb::pool_alloc(ctx, reinterpret_cast<void**>(&d), bytes, s));
    st = lrb_blr_reconstruct_dense(ctx, m, d, 1, s);
    cudaError_t e = cudaSuccess;
    if (!st) e = cudaMemcpyAsync(out, d, bytes, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (st) return st;
    if (e != cudaSuccess) return lrb::cuda_fail(ctx, e, "lrb_blr_reconstruct_dense: copy");
    if (e2 != cudaSuccess) return lrb::cuda_fail(ctx, e2, "lrb_blr_reconstruct_dense: sync");
    return LRB_OK;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  {
    const int64_t blocks = std::min<int64_t>((T * b + 7) / 8, int64_t(ctx->sm_count));
    const int vec = (b % 2 == 0 && m->pitch % 2 == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(m->d_dcat) & 15) == 0);
    // the full shared-memory carve-out, so an SM running a copy CTA can take
    // a streaming-kernel CTA (224 KB) beside it
    static const cudaError_t carve = cudaFuncSetAttribute(
        blr_diag_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    (void)carve;
    LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_diag_kernel, dim3(unsigned(blocks)), dim3(256), 0, s,
                                      m->d_dcat, out, int(T), int(b), m->pitch, vec));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (T == 1) return LRB_OK;
  // the off-diagonal tiles as one write-streaming launch (lrb_blr_recon.cu)
  // where the shape allows it; LRB_BLR_RECON=0 keeps the UX + tile-kernel form
  {
    const char* re = std::getenv("LRB_BLR_RECON");
    if (!(re && re[0] == '0') &&
        lrb::launch_blr_recon(ctx, m->d_vtcol, m->d_dcat, m->d_x, out, T, b, r, m->pitch, s, &st))
      return st;
  }
  const int64_t items = T * (T - 1);
  if (!m->d_ux) {
    size_t ux_cap = 0;
    st = grow(ctx, m, &m->d_ux, &ux_cap, size_t(items * b * r));
    if (st) return st;
  }
  using TileCfg = lrb::VariantTraits<LRB_V_Q64>::Cfg<false, false, true>;
  lrb::BlrTileProblem tp;
  std::memset(&tp, 0, sizeof(tp));
  const bool tiles_ok =
      items <= INT32_MAX &&
      lrb::encode_operand(&tp.tmA, m->d_vtcol, b, r, b, r * b, items, TileCfg::A_BOX_IN,
                          TileCfg::A_BOX_OUT) &&
      lrb::encode_operand(&tp.tmB, m->d_ux, r, b, r, b * r, items, TileCfg::B_BOX_IN,
                          TileCfg::B_BOX_OUT);
  if (!tiles_ok && m->recon_out != out) {
    // a captured graph may still execute the previous plan: retire it
    if (m->recon_plan) m->retired_plans.push_back(m->recon_plan);
    m->recon_plan = nullptr;
    m->recon_out = nullptr;
    std::vector<int64_t> mm(items, b), nn(items, b), kk(items, r), la(items, r), lb(items, b),
        lc(items, n);
    std::vector<const double*> pa(items), pb(items);
    std::vector<double*> pc(items);
    for (int64_t p = 0; p < items; ++p) {
      const int64_t j = p / (T - 1), ip = p - j * (T - 1), i = ip < j ? ip : ip + 1;
      pa[p] = m->d_ux + p * b * r;
      pb[p] = m->d_vtcol + p * r * b;
      pc[p] = out + i * b * n + j * b;
    }
    st = lrb_ptr_plan_create(ctx, 'R', 'N', 'N', items, mm.data(), nn.data(), kk.data(),
                             pa.data(), la.data(), pb.data(), lb.data(), pc.data(), lc.data(),
                             0.0, &m->recon_plan);
    if (st) return st;
    m->recon_out = out;
  }
  {
    const int64_t blocks = std::min<int64_t>(items, int64_t(ctx->sm_count) * 16);
    if (r % 8 == 0 && r <= 32 && b % 8 == 0)
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_ux_mma_kernel, dim3(unsigned(blocks)), dim3(256), 0, s,
                                        m->d_dcat, m->d_x, m->d_ux, int(T), int(b), int(r)));
    else if (r % 2 == 0)
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_ux_kernel<2>, dim3(unsigned(blocks)), dim3(256), 0, s,
                                        m->d_dcat, m->d_x, m->d_ux, int(T), int(b), int(r)));
    else
      LRB_CUDA_TRY(ctx, lrb::launch_pdl(blr_ux_kernel<1>, dim3(unsigned(blocks)), dim3(256), 0, s,
                                        m->d_dcat, m->d_x, m->d_ux, int(T), int(b), int(r)));
    ctx->launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (!tiles_ok) return lrb_ptr_plan_execute(ctx, m->recon_plan, stream);
  tp.A = m->d_vtcol;
  tp.B = m->d_ux;
  tp.C = out;
  tp.n = n;
  tp.b = int(b);
  tp.r = int(r);
  tp.tiles = int(T);
  tp.tiles_i = int((b + TileCfg::MB - 1) / TileCfg::MB);
  tp.tiles_per_item = tp.tiles_i * int((b + TileCfg::NB - 1) / TileCfg::NB);
  tp.num_tiles = items * tp.tiles_per_item;
  tp.c_tma = (r <= 16 && !(lrb::debug_flags() & 64) &&
              lrb::encode_tiles_c_map(&tp.tmC, out, n, b, TileCfg::NB))
                 ? 1
                 : 0;
  lrb::LaunchInfo info{0, 0};
  LRB_CUDA_TRY(ctx, lrb::launch_gemm<TileCfg>(tp, 0, ctx->device, ctx->sm_count, s, &info));
  if (info.grid > 0) ctx->launches.fetch_add(1, std::memory_order_relaxed);
  return LRB_OK;
}
