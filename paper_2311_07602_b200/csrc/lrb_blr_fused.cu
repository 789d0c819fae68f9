// lrb_blr_fused.cu — the BLR multi-RHS matvec (reference blr_matvec,
// proj/include/lrbatch/blr.hpp:141-175) as ONE persistent launch.
//
// The three-launch form (lrb_blr.cu: W GEMM, coupling kernel, row GEMM) pays
// two launch ramps and two wave tails on a ~0.1 ms problem, and its row step
// is a single partial wave (T x b/64 tiles on 2 x 148 slots). Here every tile
// of both GEMMs comes from one ticket sequence on one persistent grid:
//   * W tiles (column j, 64 rows of the stacked [Vt_ij]_i): W^T = rhs_j^T Vt_j^T
//     on DMMA by the four computing warps, which leave the tile in shared
//     memory with its ticket and go straight on to the next tile's chunks. A
//     sixth warp, the coupling warp, picks it up there: Z_ij = X_ij W_ij of
//     its 64 / r items (DMMA, k ascending; scalar chains at r = 4), Z written
//     into row i's operand block, then the ready count of (row i, quarter of
//     its Z columns) bumped (release). W itself is never stored.
//   * row tiles (row i, 64 columns of y_i): y_i^T = [rhs_i; Z_i*]^T [D_i|U_i*]^T
//     over K' = b + (T-1) r in ascending k; the producer streams the D_i part
//     straight from rhs and, before the first Z chunk of each quarter of row
//     i's T-1 columns, waits until that quarter's items have landed (acquire),
//     then fences the async proxy. Z columns land in ticket order (j
//     ascending), so a row tile runs most of its Z part while the last
//     columns' W tiles are still in flight.
// W tickets precede row tickets, so a waiting row tile only ever waits on
// tiles already claimed by running CTAs: progress is guaranteed. Every entry
// keeps the reference's chain order (W and Z chains over their k ascending;
// y_i's chain over D's columns, then j-major, p), so results are bitwise the
// three-launch path and the FMA-chain oracle. The last CTA out resets the
// tickets and bumps an epoch word; the ready counts only ever grow (a launch
// waits for epoch + 1 times the expected count), so graph replays need no
// memset and a launch ends without a tail of reset stores.
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "lrb_gemm.cuh"
#include "lrb_internal.h"

namespace lrb {

struct BlrFusedProblem {
  CUtensorMap tmRhs;   // rhs: (nrhs, b, T), item stride b nrhs      box (MB+4, KB)
  CUtensorMap tmVt;    // stacked Vt per column: (b, K, T)          box (KB+4, NB)
  CUtensorMap tmZ;     // Z part of rz: (nrhs, K, T), stride P nrhs box (MB+4, KB)
  CUtensorMap tmDcat;  // [D_i | U_i*] rows: (P, b, T)              box (KB+4, NB)
  const double* x;     // X_ij in (j, i) order, r x r row-major
  double* rz;          // per row i: P x nrhs, Z_ij at rows b + jp r
  double* y;           // n x nrhs row-major
  int T, b, r, nrhs, K, P;
  int ld;              // row pitch of rhs and y (>= nrhs: a column range of a wider right-hand side)
  int tw, tr;          // 64-row blocks per W column, 64-column blocks per row
  long long nw, total;  // W tiles, all tiles
  unsigned* ready;     // [T][4] Z items landed per row and quarter of its T - 1 columns
  int gs;              // columns per quarter: ceil((T - 1) / 4)
  unsigned long long* next;  // [0] tickets, [1] finished CTAs, [2] epoch (completed launches)
  int flags;           // debug probe bits (LRB_DEBUG_FLAGS)
};

namespace {

// the m16 tile, 32-deep chunks in a 4-stage ring (two CTAs per SM). Measured
// on the 16-RHS bench shape: k64 x 2 stages 0.0676 ms, k32 x 4 0.0656, k16 x
// 7 0.0697, k32 x 5 or k64 x 3 (one CTA per SM) 0.076-0.082, 32-column tiles
// 0.072-0.076
// (MBT = 16 serves 9..16 right-hand sides; MBT = 8 serves up to 8 without
// padding them to 16 rows: half the DMMA work and half the rhs / Z traffic)
template <int MBT>
using FCfgT = GemmCfg<1, 4, MBT, 16, 32, 4, 2, false, false, true>;
constexpr int kFStages = 4;
constexpr int kFWarps = 4;
constexpr int kFThreads = kFWarps * 32 + 64;  // + the producer warp + the coupling warp
constexpr int kFNB = 64, kFKB = 32;
constexpr int kMaxRank = 32;                   // ranks served (r | 64)
constexpr int kStagedRank = 16;                // up to here X_ij is staged in shared memory
constexpr int kXs = kFNB * kStagedRank;       // X tiles of one W tile: 64 / r items of r x r
// the W tile in shared memory: 64 rows of W, pitch MB + 4 doubles (the coupling
// warp's B fragments, lanes (g, tq) at tq * pitch + g, are conflict-free)
template <int MBT>
constexpr int w_pitch() { return MBT + kPad; }
template <int MBT>
constexpr size_t fused_smem() {
  // ring, the W tile (64 x nrhs), X staging, barriers + slot table + tile id
  return size_t(kFStages) * FCfgT<MBT>::STAGE_ELEMS * 8 + size_t(w_pitch<MBT>() * kFNB) * 8 +
         size_t(kXs) * 8 + size_t(kFStages) * 8 * 3 + 48;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

template <int MBT>
__global__ void __launch_bounds__(kFThreads, 2)
    blr_fused_kernel(const __grid_constant__ BlrFusedProblem p) {
  using FCfg = FCfgT<MBT>;
  static_assert(FCfg::STAGES == kFStages && FCfg::NB == kFNB && FCfg::KB == kFKB, "ring geometry");
  constexpr int WP = w_pitch<MBT>();
  constexpr int kScratch = WP * FCfg::NB;
  pdl_entry();
  constexpr int KB = FCfg::KB, NB = FCfg::NB, MB = FCfg::MB;
  extern __shared__ __align__(1024) double smem[];
  double* scratch = smem + size_t(kFStages) * FCfg::STAGE_ELEMS;
  double* xs = scratch + kScratch;  // the W tile's X_ij (bulk copy by the producer)
  uint64_t* full = reinterpret_cast<uint64_t*>(xs + kXs);
  uint64_t* empty = full + kFStages;
  volatile long long* slot = reinterpret_cast<volatile long long*>(empty + kFStages);
  // W tile hand-over to the coupling warp: xfull (the producer's bulk copy
  // of the tile's X_ij landed), wfull (the computing warps have written the
  // W tile and its ticket), cfree (the coupling warp is done with both)
  uint64_t* xfull = reinterpret_cast<uint64_t*>(const_cast<long long*>(slot + kFStages));
  uint64_t* wfull = xfull + 1;
  uint64_t* cfree = xfull + 2;
  volatile long long* ctile = reinterpret_cast<volatile long long*>(xfull + 3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kFWarps);
    }
    mbar_init(xfull, 1);
    mbar_init(wfull, kFWarps * 32);
    mbar_init(cfree, 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kFWarps) {  // the producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      long long q = 0;
      long long nwt = 0;  // W tiles issued (X staging parity)
      // (bit 8: streaming probe, wrong results — no rhs / Z operand loads)
      const bool no_a = (p.flags & 256) != 0;
      const uint32_t bytes = (uint32_t(no_a ? 0 : FCfg::A_BOX) + uint32_t(FCfg::B_BOX)) * 8u;
      const uint64_t pol_stream = policy_evict_normal(), pol_keep = policy_evict_last();
      // (bits 10 / 11: phase probes, wrong results — W tiles only / row tiles only)
      const long long t_off = (p.flags & 2048) ? p.nw : 0;
      const long long t_end = (p.flags & 1024) ? p.nw : p.total;
      // the first ticket is the CTA's own index: 296 CTAs claiming from one
      // word at launch would queue behind each other at the L2 (same-address
      // atomics serialise); the ticket word then counts from gridDim.x
      const long long t_dyn = t_off + gridDim.x;
      long long t = t_off + blockIdx.x;
      // (bit 3: probe, claim the next tile while this one's first chunk is in
      // flight; measured slower: a CTA busy on a long row tile then holds a
      // ticket other CTAs could start)
      const bool ahead = (p.flags & 8) != 0;
      const unsigned long long epoch = p.next[2];  // launches completed on these sync words
      // (bit 1: probe, wait for every quarter of Z_i* before the first Z chunk)
      const bool all_first = (p.flags & 2) != 0;
#pragma unroll 1
      while (true) {
        if (q >= kFStages) mbar_wait(&empty[stage], phase ^ 1);
        if (t >= t_end) {
          slot[stage] = -1;
          mbar_arrive(&full[stage]);
          break;
        }
        const bool wtile = t < p.nw;
        const long long u = wtile ? t : t - p.nw;
        // W tickets run column-major (all of column j's blocks, then column
        // j + 1). Bit 6 probes the row-block-major order (every column's block
        // 0 first, so the early rows' Z are complete long before the first row
        // tickets): no change on the 16-RHS shape, 2.5 % slower on the paper's
        // 8-RHS shape (a column's tiles share rhs_j in L2).
        const bool colmajor = (p.flags & 64) == 0;
        const int z = int(wtile ? (colmajor ? u / p.tw : u % p.T) : u / p.tr);  // column j / row i
        const int n0 = int(wtile ? (colmajor ? u % p.tw : u / p.T) : u % p.tr) * NB;
        const int kend = wtile ? p.b : p.P;
        int grp = 0;  // quarters of row z's Z columns known to have landed
        int zk = p.b;  // first k of quarter grp's Z rows
        long long t_next = -1;
#pragma unroll 1
        for (int k0 = 0; k0 < kend; k0 += KB) {
          if (k0 > 0 && q >= kFStages) mbar_wait(&empty[stage], phase ^ 1);
          const void* mapA = &p.tmRhs;
          int ka = k0;
          if (!wtile && k0 >= p.b) {
            // Z_i* lands from the W tiles' coupling, column j ascending like
            // the tickets: wait (acquire) only for the quarters of columns
            // this chunk reaches, so a row tile starts its Z part while the
            // last columns' W tiles are still running
            if (grp < 4 && (all_first || k0 + KB > zk)) {
              do {
                const unsigned want =
                    (unsigned(epoch) + 1u) * unsigned(min(p.gs, p.T - 1 - grp * p.gs));
                while (!(p.flags & 32) &&
                       int(ld_acquire_u32(&p.ready[z * 4 + grp]) - want) < 0)
                  __nanosleep(64);  // (bit 5: probe, no wait: wrong results)
                ++grp;
                zk += p.gs * p.r;  // first k of the next quarter's Z rows
              } while (grp < 4 && (all_first || k0 + KB > zk) && zk < kend);
              if (zk >= kend) grp = 4;
              fence_proxy_async_global();
            }
            mapA = &p.tmZ;
            ka = k0 - p.b;
          }
          slot[stage] = t;
          fence_proxy_async_smem();
          double* As = smem + size_t(stage) * FCfg::STAGE_ELEMS;
          double* Bs = As + FCfg::A_ELEMS;
          mbar_arrive_expect_tx(&full[stage], bytes);
          if (!no_a) tma_load_3d(As, mapA, 0, ka, z, &full[stage], pol_keep);
          if (wtile)
            tma_load_3d(Bs, &p.tmVt, k0, n0, z, &full[stage], pol_stream);
          else
            tma_load_3d(Bs, &p.tmDcat, k0, n0, z, &full[stage], pol_stream);
          ++q;
          if (++stage == kFStages) {
            stage = 0;
            phase ^= 1;
          }
          if (k0 == 0 && ahead && wtile)
            t_next = static_cast<long long>(atomicAdd(p.next, 1ull)) + t_dyn;
        }
        if (wtile && p.r <= kStagedRank) {
          // the tile's X_ij (items ip0 .. of column j are consecutive in
          // (j, i) order: one contiguous bulk copy), issued after the tile's
          // chunks: by now the coupling warp has finished the previous W
          // tile and released xs
          if (nwt > 0) mbar_wait(cfree, uint32_t((nwt - 1) & 1));
          const int items = min(NB, p.K - n0) / p.r;
          const uint32_t xb = uint32_t(items) * p.r * p.r * 8u;
          mbar_arrive_expect_tx(xfull, xb);
          bulk_g2s(xs, p.x + (int64_t(z) * (p.T - 1) + n0 / p.r) * p.r * p.r, xb, xfull,
                   pol_stream);
          ++nwt;
        }
        t = (ahead && wtile) ? t_next : static_cast<long long>(atomicAdd(p.next, 1ull)) + t_dyn;
      }
      // the last CTA out resets the tickets and opens the next epoch (the
      // ready counts are never reset: no tail of stores at the end of a launch)
      __threadfence();
      const unsigned long long done = atomicAdd(p.next + 1, 1ull);
      if (done == gridDim.x - 1) {
        p.next[0] = 0;
        p.next[1] = 0;
        p.next[2] = epoch + 1;
        __threadfence();
      }
    }
    return;
  }

  const int g = lane >> 2, tq = lane & 3;
  if (warp == kFWarps + 1) {
    // The coupling warp: Z_ij = X_ij W_ij for the items of each W tile this
    // CTA computes, off the computing warps' path (they go straight on to the
    // next tile's chunks). Z goes into row i's operand block, then row i's
    // ready count is bumped (release).
    long long nwc = 0;  // W tiles handled (barrier parity)
#pragma unroll 1
    while (true) {
      mbar_wait(wfull, uint32_t(nwc & 1));
      const long long t = *ctile;
      if (t < 0) break;
      const bool colmajor = (p.flags & 64) == 0;
      const int jcol = int(colmajor ? t / p.tw : t % p.T);
      const int n0 = int(colmajor ? t % p.tw : t / p.T) * NB;
      const int r = p.r, nrhs = p.nrhs;
      const int items = min(NB, p.K - n0) / r;
      const int ip0 = n0 / r;
      if (r <= kStagedRank) mbar_wait(xfull, uint32_t(nwc & 1));  // this tile's X_ij landed
      ++nwc;
      if (p.flags & 16) {
        // (bit 4: probe, no coupling)
      } else if (r == 32) {
        // rank 32: the tile's two X_ij do not fit beside the ring, so the
        // fragments come straight from global memory (read once; all of an
        // item's loads are in flight before its chains start). Same 8x8
        // blocks, k ascending in steps of 4.
        for (int it = 0; it < items; ++it) {
          const int ip = ip0 + it;
          const int i = ip < jcol ? ip : ip + 1;
          const int jp = jcol < i ? jcol : jcol - 1;
          double* zrow = p.rz + (int64_t(i) * p.P + p.b + int64_t(jp) * 32) * nrhs;
          const double* xg = p.x + (int64_t(jcol) * (p.T - 1) + ip) * 1024;
          const double* wt = scratch + it * 32 * WP;
          constexpr int CN = MB / 8;
          double a[4][8];
#pragma unroll
          for (int pi = 0; pi < 4; ++pi)
#pragma unroll
            for (int kq = 0; kq < 8; ++kq) a[pi][kq] = __ldg(xg + (pi * 8 + g) * 32 + kq * 4 + tq);
          double d[4][CN][2];
#pragma unroll
          for (int pi = 0; pi < 4; ++pi)
#pragma unroll
            for (int ci = 0; ci < CN; ++ci) d[pi][ci][0] = d[pi][ci][1] = 0.0;
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) {
            double bv[CN];
#pragma unroll
            for (int ci = 0; ci < CN; ++ci) bv[ci] = wt[(kq * 4 + tq) * WP + ci * 8 + g];
#pragma unroll
            for (int pi = 0; pi < 4; ++pi)
#pragma unroll
              for (int ci = 0; ci < CN; ++ci)
                dmma_8x8x4(d[pi][ci][0], d[pi][ci][1], a[pi][kq], bv[ci]);
          }
#pragma unroll
          for (int pi = 0; pi < 4; ++pi)
#pragma unroll
            for (int ci = 0; ci < CN; ++ci) {
              const int c = ci * 8 + 2 * tq;
              double* zp = zrow + int64_t(pi * 8 + g) * nrhs + c;
              if (c + 1 < nrhs)
                *reinterpret_cast<double2*>(zp) = make_double2(d[pi][ci][0], d[pi][ci][1]);
              else if (c < nrhs)
                *zp = d[pi][ci][0];
            }
        }
      } else if (r % 8 == 0) {
        // DMMA: 8x8 output blocks, k ascending in steps of 4 (each entry one
        // in-order FMA chain). W columns nrhs..MB-1 are zero (TMA fills the
        // rhs box past its extent) and are not stored.
        for (int it = 0; it < items; ++it) {
          const int ip = ip0 + it;
          const int i = ip < jcol ? ip : ip + 1;
          const int jp = jcol < i ? jcol : jcol - 1;
          double* zrow = p.rz + (int64_t(i) * p.P + p.b + int64_t(jp) * r) * nrhs;
          constexpr int CN = MB / 8;
          double d[2][CN][2];
#pragma unroll
          for (int pi = 0; pi < 2; ++pi)
#pragma unroll
            for (int ci = 0; ci < CN; ++ci) d[pi][ci][0] = d[pi][ci][1] = 0.0;
          const double* xi = xs + it * r * r;
          const double* wt = scratch + it * r * WP;
          const bool two = r > 8;  // r in {8, 16}
          // all fragment loads of the item first, then the chains
          double a[2][4], bv[CN][4];
#pragma unroll
          for (int kq = 0; kq < 4; ++kq) {
            const int k = min(kq * 4 + tq, r - 1);  // (r = 8: steps 2, 3 are not used)
            a[0][kq] = xi[g * r + k];
            a[1][kq] = two ? xi[(8 + g) * r + k] : 0.0;
#pragma unroll
            for (int ci = 0; ci < CN; ++ci) bv[ci][kq] = wt[k * WP + ci * 8 + g];
          }
#pragma unroll
          for (int kq = 0; kq < 4; ++kq) {
            if (kq * 4 < r) {
#pragma unroll
              for (int ci = 0; ci < CN; ++ci) {
                dmma_8x8x4(d[0][ci][0], d[0][ci][1], a[0][kq], bv[ci][kq]);
                if (two) dmma_8x8x4(d[1][ci][0], d[1][ci][1], a[1][kq], bv[ci][kq]);
              }
            }
          }
#pragma unroll
          for (int pi = 0; pi < 2; ++pi) {
            if (pi == 1 && !two) break;
#pragma unroll
            for (int ci = 0; ci < CN; ++ci) {
              const int c = ci * 8 + 2 * tq;
              double* zp = zrow + int64_t(pi * 8 + g) * nrhs + c;
              if (c + 1 < nrhs)
                *reinterpret_cast<double2*>(zp) = make_double2(d[pi][ci][0], d[pi][ci][1]);
              else if (c < nrhs)
                *zp = d[pi][ci][0];
            }
          }
        }
      } else {
        // scalar chains (r = 4): one Z entry per lane and round, k ascending
        const int per = r * nrhs, total = items * per;
        for (int e = lane; e < total; e += 32) {
          const int it = e / per, rem = e - it * per;
          const int pr = rem / nrhs, cc = rem - pr * nrhs;
          const double* xr = xs + (it * r + pr) * r;
          const double* wc = scratch + it * r * WP + cc;
          double zacc = 0.0;
          for (int k = 0; k < r; ++k) zacc = fma(xr[k], wc[k * WP], zacc);
          const int ip = ip0 + it;  // row index i' of column j's stack
          const int i = ip < jcol ? ip : ip + 1;
          const int jp = jcol < i ? jcol : jcol - 1;
          p.rz[(int64_t(i) * p.P + p.b + int64_t(jp) * r + pr) * nrhs + cc] = zacc;
        }
      }
      // release: the warp barrier orders every lane's Z stores before the
      // counting lanes' fences (cumulativity), so only those lanes fence
      __syncwarp();
      if (lane == 0) mbar_arrive(cfree);  // xs and the W tile may be refilled
      if (lane < items) {
        const int ip = ip0 + lane;
        const int i = ip < jcol ? ip : ip + 1;
        const int jp = jcol < i ? jcol : jcol - 1;
        __threadfence();
        atomicAdd(&p.ready[i * 4 + jp / p.gs], 1u);
      }
    }
    return;
  }

  const int wi = 0, wj = warp;
  int stage = 0;
  uint32_t phase = 0;
  long long nwm = 0;  // W tiles handed to the coupling warp (barrier parity)
#pragma unroll 1
  while (true) {
    mbar_wait(&full[stage], phase);
    const long long t = slot[stage];
    if (t < 0) {  // tell the coupling warp too
      if (nwm > 0) mbar_wait(cfree, uint32_t((nwm - 1) & 1));
      if (threadIdx.x == 0) *ctile = -1;
      mbar_arrive(wfull);
      break;
    }
    const bool wtile = t < p.nw;
    const long long u = wtile ? t : t - p.nw;
    const bool colmajor = (p.flags & 64) == 0;
    const int z = int(wtile ? (colmajor ? u / p.tw : u % p.T) : u / p.tr);
    const int n0 = int(wtile ? (colmajor ? u % p.tw : u / p.T) : u % p.tr) * NB;
    const int chunks = ((wtile ? p.b : p.P) + KB - 1) / KB;
    double acc[FCfg::FJ][FCfg::FI][2];
#pragma unroll
    for (int fj = 0; fj < FCfg::FJ; ++fj)
#pragma unroll
      for (int fi = 0; fi < FCfg::FI; ++fi) acc[fj][fi][0] = acc[fj][fi][1] = 0.0;
#pragma unroll 1
    for (int c = 0; c < chunks; ++c) {
      if (c > 0) mbar_wait(&full[stage], phase);
      const double* As = smem + size_t(stage) * FCfg::STAGE_ELEMS;
      const double* Bs = As + FCfg::A_ELEMS;
      // a partial last chunk is zero-filled by TMA: +0 terms leave the chains exact
      if (!(p.flags & 128)) {  // (bit 7: probe, no products)
#pragma unroll
        for (int kq = 0; kq < KB / 4; ++kq) mma_kstep<FCfg>(acc, As, Bs, wi, wj, g, kq * 4 + tq);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kFStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (!wtile) {
      // y_i rows n0.. : C^T(c, j) -> y[(i b + n0 + j) nrhs + c]
      const int i = z;
#pragma unroll
      for (int fj = 0; fj < FCfg::FJ; ++fj) {
        const int j = n0 + FCfg::load_col(wj, fj, g);
        if (j >= p.b) continue;
        double* yr = p.y + (int64_t(i) * p.b + j) * p.ld;
        const int c0 = FCfg::acc_row(wi, 0, 0, tq);
        if constexpr (FCfg::FI == 2) {  // paired fragments: rows c0 .. c0 + 3
          const double v[4] = {acc[fj][0][0], acc[fj][1][0], acc[fj][0][1], acc[fj][1][1]};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (c0 + e < p.nrhs) yr[c0 + e] = v[e];
        } else {  // rows c0, c0 + 1
          if (c0 < p.nrhs) yr[c0] = acc[fj][0][0];
          if (c0 + 1 < p.nrhs) yr[c0 + 1] = acc[fj][0][1];
        }
      }
      continue;
    }
    // W tile: W rows into shared memory (scratch[j * WP + c] = W(n0 + j, c))
    // with the ticket, handed to the coupling warp; the computing warps go on
    if (nwm > 0) mbar_wait(cfree, uint32_t((nwm - 1) & 1));  // the previous W tile is consumed
    ++nwm;
#pragma unroll
    for (int fj = 0; fj < FCfg::FJ; ++fj) {
      const int j = FCfg::load_col(wj, fj, g);
      const int c0 = FCfg::acc_row(wi, 0, 0, tq);
      if constexpr (FCfg::FI == 2) {
        scratch[j * WP + c0 + 0] = acc[fj][0][0];
        scratch[j * WP + c0 + 1] = acc[fj][1][0];
        scratch[j * WP + c0 + 2] = acc[fj][0][1];
        scratch[j * WP + c0 + 3] = acc[fj][1][1];
      } else {
        scratch[j * WP + c0 + 0] = acc[fj][0][0];
        scratch[j * WP + c0 + 1] = acc[fj][0][1];
      }
    }
    if (threadIdx.x == 0) *ctile = u;
    mbar_arrive(wfull);
  }
}

}  // namespace

bool encode_operand(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                    int64_t stride, int64_t zdim, int box_in, int box_out);

// One fused matvec launch, or false (nothing launched) when the shape is
// outside what the fused kernel serves: nrhs <= 16, block a multiple of 32,
// rank dividing 64 (each 64-row W block holds whole items) and a multiple of
// 4, TMA-addressable operands.
template <int MBT>
bool launch_blr_fused_t(lrb_ctx* ctx, const double* rhs, int64_t nrhs, int64_t ld, double* y,
                        int64_t T,
                        int64_t b, int64_t r, int64_t P, const double* vtcol, const double* x,
                        const double* dcat, double* rz, unsigned* ready,
                        unsigned long long* next, cudaStream_t s, lrb_status* st) {
  using FCfg = FCfgT<MBT>;
  constexpr size_t kFSmem = fused_smem<MBT>();
  const int64_t K = (T - 1) * r;
  BlrFusedProblem p;
  std::memset(&p, 0, sizeof(p));
  const bool ok =
      encode_operand(&p.tmRhs, rhs, nrhs, b, ld, b * ld, T, FCfg::MB + kPad, FCfg::KB) &&
      encode_operand(&p.tmVt, vtcol, b, K, b, K * b, T, FCfg::KB + kPad, FCfg::NB) &&
      encode_operand(&p.tmZ, rz + b * nrhs, nrhs, K, nrhs, P * nrhs, T, FCfg::MB + kPad,
                     FCfg::KB) &&
      encode_operand(&p.tmDcat, dcat, P, b, P, b * P, T, FCfg::KB + kPad, FCfg::NB);
  if (!ok) return false;
  p.x = x;
  p.rz = rz;
  p.y = y;
  p.T = int(T), p.b = int(b), p.r = int(r), p.nrhs = int(nrhs), p.K = int(K), p.P = int(P);
  p.ld = int(ld);
  p.tw = int((K + FCfg::NB - 1) / FCfg::NB);
  p.tr = int((b + FCfg::NB - 1) / FCfg::NB);
  p.nw = int64_t(T) * p.tw;
  p.total = p.nw + int64_t(T) * p.tr;
  p.ready = ready;
  p.gs = int((T - 1 + 3) / 4);
  p.next = next;
  p.flags = debug_flags();
  static int occ_cache[64] = {0};
  const int dev = ctx->device;
  int occ = (dev >= 0 && dev < 64) ? occ_cache[dev] : 0;
  cudaError_t e = cudaSuccess;
  if (occ == 0) {
    e = cudaFuncSetAttribute(blr_fused_kernel<MBT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kFSmem));
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, blr_fused_kernel<MBT>, kFThreads,
                                                        kFSmem);
    if (e == cudaSuccess && occ < 1) e = cudaErrorInvalidConfiguration;
    if (e == cudaSuccess && dev >= 0 && dev < 64) occ_cache[dev] = occ;
  }
  if (e == cudaSuccess) {
    const int64_t grid = std::min<int64_t>(int64_t(ctx->sm_count) * occ, p.total);
    e = launch_pdl(blr_fused_kernel<MBT>, dim3(unsigned(grid)), dim3(kFThreads), kFSmem, s, p);
  }
  if (e != cudaSuccess) {
    *st = cuda_fail(ctx, e, "blr_fused_kernel launch");
    return true;
  }
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  *st = LRB_OK;
  return true;
}

// the shapes the fused kernel serves (its operands must be TMA-addressable too)
bool blr_fused_shape_ok(int64_t T, int64_t b, int64_t r, int64_t nrhs) {
  return T >= 2 && nrhs >= 1 && nrhs <= 16 && r >= 4 && b % kFKB == 0 && kFNB % r == 0 &&
         r % 4 == 0 && r <= kMaxRank;
}

bool launch_blr_fused(lrb_ctx* ctx, const double* rhs, int64_t nrhs, int64_t ld, double* y,
                      int64_t T,
                      int64_t b, int64_t r, int64_t P, const double* vtcol, const double* x,
                      const double* dcat, double* rz, unsigned* ready,
                      unsigned long long* next, cudaStream_t s, lrb_status* st) {
  if (!blr_fused_shape_ok(T, b, r, nrhs)) return false;
  if (nrhs <= 8) {
    // the m8 tile; LRB_BLR_FUSED_M8=0 keeps the three-launch form for <= 8
    // right-hand sides
    const char* e8 = std::getenv("LRB_BLR_FUSED_M8");
    if (e8 && e8[0] == '0') return false;
    return launch_blr_fused_t<8>(ctx, rhs, nrhs, ld, y, T, b, r, P, vtcol, x, dcat, rz, ready, next, s,
                                 st);
  }
  return launch_blr_fused_t<16>(ctx, rhs, nrhs, ld, y, T, b, r, P, vtcol, x, dcat, rz, ready, next, s,
                                st);
}

}  // namespace lrb
