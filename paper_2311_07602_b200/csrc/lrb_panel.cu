// lrb_panel.cu — the row-panel kernel for short-k products (k <= 32): the
// low-rank expansion C_i = U_i * V_i^T (BASELINE cfg2; reference
// blr.hpp:75-78 reconstruct U·Vt, dense.hpp:43-56 per item).
//
// Why a second kernel. At k = 32 every 64 x 64 tile of the general kernel
// (lrb_gemm.cuh) is only 8 DMMA k-steps long, so its per-tile overhead is not
// amortised, and the C write stream (89% of cfg2's bytes) evicts the U / V
// panels the neighbouring tiles still need from L2: cfg2 reads 1.8-3.1x its
// algorithmic operand bytes from DRAM (profiles/). Here:
//   * A unit is (item, 256-row block). Its U panel (256 x k) lands in shared
//     memory once (two 132-row TMA boxes, pitch 132: conflict-free fragment
//     loads) and stays there while all of V streams past it, double-buffered
//     across units. V streams in 32-column chunks through an 8-slot ring. The
//     operands therefore leave DRAM about once, whatever the C stream does
//     to L2.
//   * Eight MMA warps (two warpgroups, 2 warps per SM sub-partition) and a
//     third warpgroup whose first warp issues every TMA load (U panels, V
//     chunks) behind full / empty mbarriers. setmaxnreg moves the producer
//     warpgroup's registers to the MMA warpgroups (40 / 232 per thread): a
//     plain ninth warp caps everyone at 168 and the 64 x 32 slabs spill
//     (cfg2 0.56). Against the self-refilling eight-warp form (the last warp
//     to release a V slot or U buffer issues its refill, kept behind
//     LRB_PANEL_PROD=0): cfg2 0.911 -> 0.918, store-free probe 0.948 -> 0.959.
//   * The producer form also splits the last round of units: its rem units
//     are cut into column ranges over rem * split CTAs, so the wave tail
//     costs 1 / split of a unit (cfg2: 55 rounds + 52 units, split in 2;
//     0.918 -> 0.924).
//   * The MMA warps form two groups of four. Group g takes the chunks of
//     parity g: each warp owns a 64 x 32 slab of the chunk's 256 x 32 C tile
//     (64 accumulators, 256 DMMAs per chunk at k = 32), and the groups run
//     free, so one group's MMAs cover the other's epilogue. Measured
//     alternatives (cfg2, fraction of FP64 peak): strict turns on the tensor
//     pipe through named barriers 0.88 (free: 0.91); splitting each slab into
//     two row halves so one half's stores interleave with the other half's
//     MMAs 0.79-0.81 (16 accumulators per phase, and the stores between
//     k-steps break the fragment-load schedule).
// Arithmetic is the general kernel's: DMMA 8x8x4 k-steps in ascending k and a
// scalar fma() tail, so every C entry is the reference's in-order FMA chain.
#include "lrb_gemm.cuh"
#include "lrb_panel.h"

namespace lrb {

namespace {

// producer form: registers per thread after setmaxnreg (MMA warpgroups,
// producer warpgroup): 2 x 128 x 232 + 128 x 40 = 64.5K of the SM's 64K
constexpr int kPanelMmaRegs = 232, kPanelProdRegs = 40;

template <bool B_T, bool PROD = false>
struct PanelCfg {
  // one MMA warp's view: a 128-row half panel (pitch 132) times a 32-column
  // chunk, warp tile 64 x 32 (GemmCfg supplies the fragment maps and offsets)
  using W = GemmCfg<2, 1, 64, 32, 32, 2, 1, false, B_T, true>;
  static constexpr int ROWS = kPanelRows;  // C rows per unit
  static constexpr int COLS = W::NB;       // C columns per chunk
  static constexpr int KMAX = W::KB;
  static constexpr int S = kPanelStages;
  static constexpr int HALF = W::A_ELEMS;  // one 132 x 32 half panel
  static constexpr int U_ELEMS = 2 * HALF;
  static constexpr int V_ELEMS = W::B_ELEMS;
  static constexpr int MMA_WARPS = 8;
  // PROD: a third warpgroup whose first warp issues every TMA load;
  // setmaxnreg moves its registers to the two MMA warpgroups
  static constexpr int THREADS = MMA_WARPS * 32 + (PROD ? 128 : 0);
  static constexpr size_t SMEM_BYTES = (size_t(2) * U_ELEMS + size_t(S) * V_ELEMS) * 8 +
                                       size_t(2 + S) * 8 * (PROD ? 2 : 1) + size_t(2 + S) * 4 + 8;
  static_assert(W::MB * 2 == ROWS, "two half panels per unit");
  static_assert(S % 2 == 0, "a slot must always feed the same group");
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// Issue unit lu's U panel (both half boxes) into buffer lu & 1 (one lane).
template <class P>
__device__ __forceinline__ void issue_panel(const StridedProblem& prob, double* U, uint64_t* u_full,
                                            int64_t lu, int units_per_item) {
  using W = typename P::W;
  const int64_t u = blockIdx.x + lu * gridDim.x;
  const int64_t item = u / units_per_item;
  const int i0 = int(u - item * units_per_item) * P::ROWS;
  const int za = prob.a_batched ? int(item) : 0;
  const int b = int(lu & 1);
  double* ub = U + b * P::U_ELEMS;
  // U is read by this unit only
  const uint64_t pol = policy_evict_normal();
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&u_full[b], uint32_t(2 * W::A_BOX) * 8u);
  tma_load_3d(ub, &prob.tmA, i0, 0, za, &u_full[b], pol);
  tma_load_3d(ub + P::HALF, &prob.tmA, i0 + W::MB, 0, za, &u_full[b], pol);
}

// Producer form: unit u's U panel into buffer b, and chunk c of unit u into
// slot s (one lane)
template <class P>
__device__ __forceinline__ void issue_panel_u(const StridedProblem& prob, double* U,
                                              uint64_t* u_full, int b, int64_t u,
                                              int units_per_item) {
  using W = typename P::W;
  const int64_t item = u / units_per_item;
  const int i0 = int(u - item * units_per_item) * P::ROWS;
  const int za = prob.a_batched ? int(item) : 0;
  double* ub = U + b * P::U_ELEMS;
  const uint64_t pol = policy_evict_normal();
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&u_full[b], uint32_t(2 * W::A_BOX) * 8u);
  tma_load_3d(ub, &prob.tmA, i0, 0, za, &u_full[b], pol);
  tma_load_3d(ub + P::HALF, &prob.tmA, i0 + W::MB, 0, za, &u_full[b], pol);
}
template <class P, bool B_T>
__device__ __forceinline__ void issue_chunk_u(const StridedProblem& prob, double* V,
                                              uint64_t* v_full, int s, int64_t u, int c,
                                              int units_per_item) {
  using W = typename P::W;
  const int64_t item = u / units_per_item;
  const int zb = prob.b_batched ? int(item) : 0;
  double* vs = V + s * P::V_ELEMS;
  const uint64_t pol = units_per_item > 1 ? policy_evict_last() : policy_evict_normal();
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&v_full[s], uint32_t(W::B_BOX) * 8u);
  if (B_T)
    tma_load_3d(vs, &prob.tmB, c * P::COLS, 0, zb, &v_full[s], pol);
  else
    tma_load_3d(vs, &prob.tmB, 0, c * P::COLS, zb, &v_full[s], pol);
}

// Issue chunk q (the CTA's q-th 32-column V chunk) into slot q % S (one lane).
template <class P, bool B_T>
__device__ __forceinline__ void issue_chunk_v(const StridedProblem& prob, double* V,
                                              uint64_t* v_full, int64_t q, int chunks,
                                              int units_per_item) {
  using W = typename P::W;
  const int64_t lu = q / chunks;
  const int c = int(q - lu * chunks);
  const int64_t u = blockIdx.x + lu * gridDim.x;
  const int64_t item = u / units_per_item;
  const int zb = prob.b_batched ? int(item) : 0;
  const int s = int(q % P::S);
  double* vs = V + s * P::V_ELEMS;
  // V is read by every unit of its item: evict-last while there are several
  const uint64_t pol = units_per_item > 1 ? policy_evict_last() : policy_evict_normal();
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&v_full[s], uint32_t(W::B_BOX) * 8u);
  if (B_T)
    tma_load_3d(vs, &prob.tmB, c * P::COLS, 0, zb, &v_full[s], pol);
  else
    tma_load_3d(vs, &prob.tmB, 0, c * P::COLS, zb, &v_full[s], pol);
}

template <bool B_T, bool PROD>
__global__ void __launch_bounds__(PanelCfg<B_T, PROD>::THREADS, 1)
    lrb_panel_kernel(const __grid_constant__ StridedProblem prob, const int flags) {
  using P = PanelCfg<B_T, PROD>;
  using W = typename P::W;
  constexpr int S = P::S, FI = W::FI, FJ = W::FJ;
  // flags bit 0: beta = 1; debug probe bit 1 skips the C stores
  const int beta_one = flags & 1;
  pdl_entry();
  extern __shared__ __align__(1024) double smem[];
  double* const U = smem;                    // [2 buffers][2 halves][HALF]
  double* const V = smem + 2 * P::U_ELEMS;   // [S][V_ELEMS]
  uint64_t* const bars = reinterpret_cast<uint64_t*>(V + S * P::V_ELEMS);
  uint64_t* const u_full = bars;             // [2]
  uint64_t* const v_full = bars + 2;         // [S]
  int* const u_rel = reinterpret_cast<int*>(bars + 2 + S);  // [2] warps past the unit
  int* const v_rel = u_rel + 2;                              // [S] warps past the chunk
  // producer form: empty barriers after the counters (8-byte aligned)
  uint64_t* const u_empty = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(v_rel + S) + 7) & ~uintptr_t(7));
  uint64_t* const v_empty = u_empty + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m = prob.m, n = prob.n, k = prob.k;
  const int units_per_item = (m + P::ROWS - 1) / P::ROWS;
  const int chunks = (n + P::COLS - 1) / P::COLS;
  const int64_t num_units = prob.num_tiles;  // host: units_per_item * batch
  const int64_t my_units =
      blockIdx.x < num_units ? (num_units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t q_total = my_units * chunks;
  // Producer form: when the last round of units would leave most CTAs idle,
  // its rem units are split into column ranges over rem * split CTAs (cfg2:
  // 8192 units on 148 CTAs = 55 rounds + 52 units, split in 2)
  int64_t n_full = my_units, part_unit = -1;
  int part_lo = 0, part_hi = 0;
  if (PROD) {
    const int64_t G = gridDim.x, rounds = num_units / G, rem = num_units - rounds * G;
    const int64_t split = rem > 0 ? min(int64_t(chunks), G / rem) : 1;
    if (split >= 2) {
      n_full = rounds;
      if (blockIdx.x < rem * split) {
        const int64_t pu = blockIdx.x / split, part = blockIdx.x - pu * split;
        part_unit = rounds * G + pu;
        part_lo = int(part * chunks / split);
        part_hi = int((part + 1) * chunks / split);
      }
    }
  }
  const int64_t n_items = n_full + (part_unit >= 0 ? 1 : 0);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      mbar_init(&u_full[b], 1);
      u_rel[b] = 0;
      if (PROD) mbar_init(&u_empty[b], P::MMA_WARPS);
    }
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      mbar_init(&v_full[s], 1);
      v_rel[s] = 0;
      if (PROD) mbar_init(&v_empty[s], P::MMA_WARPS / 2);
    }
    fence_mbar_init();
    if (!PROD) {
      // prologue: the first two U panels and the first S chunks
      for (int64_t lu = 0; lu < 2 && lu < my_units; ++lu)
        issue_panel<P>(prob, U, u_full, lu, units_per_item);
      for (int64_t q = 0; q < S && q < q_total; ++q)
        issue_chunk_v<P, B_T>(prob, V, v_full, q, chunks, units_per_item);
    }
  }
  __syncthreads();
  if constexpr (PROD) {
    if (warp >= P::MMA_WARPS) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kPanelProdRegs));
      // producer: U panels and V chunks in consumption order behind the
      // empty barriers
      if (warp == P::MMA_WARPS && lane == 0) {
        int64_t q = 0;
#pragma unroll 1
        for (int64_t lu = 0; lu < n_items; ++lu) {
          const bool full = lu < n_full;
          const int64_t u = full ? blockIdx.x + lu * gridDim.x : part_unit;
          if (lu >= 2) mbar_wait(&u_empty[lu & 1], int((lu >> 1) - 1) & 1);
          issue_panel_u<P>(prob, U, u_full, int(lu & 1), u, units_per_item);
          const int hi = full ? chunks : part_hi;
#pragma unroll 1
          for (int c = full ? 0 : part_lo; c < hi; ++c, ++q) {
            if (q >= S) mbar_wait(&v_empty[q % S], int(q / S - 1) & 1);
            issue_chunk_u<P, B_T>(prob, V, v_full, int(q % S), u, c, units_per_item);
          }
        }
      }
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kPanelMmaRegs));
  }

  // -------------------------------------------------------------- MMA warps
  const int grp = warp >> 2;       // chunk parity this warp's group takes
  const int slab = warp & 3;       // 64-row slab of the 256-row unit
  const int half = slab >> 1;      // which 128-row half panel
  const int wi = slab & 1;         // 64-row warp tile inside the half
  const int g = lane >> 2, tq = lane & 3;

  int64_t q = 0;
#pragma unroll 1
  for (int64_t lu = 0; lu < n_items; ++lu) {
    const bool full_unit = lu < n_full;
    const int64_t u = full_unit ? blockIdx.x + lu * gridDim.x : part_unit;
    const int64_t item = u / units_per_item;
    const int i0 = int(u - item * units_per_item) * P::ROWS + half * W::MB;  // this half's row 0
    double* const Cb = prob.C + item * prob.sC;
    const int b = int(lu & 1);
    mbar_wait(&u_full[b], int(lu >> 1) & 1);
    const double* As = U + b * P::U_ELEMS + half * P::HALF;
    const int c_hi = full_unit ? chunks : part_hi;
#pragma unroll 1
    for (int c = full_unit ? 0 : part_lo; c < c_hi; ++c, ++q) {
      if (int(q & 1) != grp) continue;
      const int s = int(q % S);
      const int j0 = c * P::COLS;
      const bool vec4_ok =
          ((reinterpret_cast<uintptr_t>(Cb) & 31) == 0) && ((prob.ldc & 3) == 0);

      double acc[FJ][FI][2];
#pragma unroll
      for (int fj = 0; fj < FJ; ++fj)
#pragma unroll
        for (int fi = 0; fi < FI; ++fi) acc[fj][fi][0] = acc[fj][fi][1] = 0.0;
      if (beta_one) {
#pragma unroll
        for (int fj = 0; fj < FJ; ++fj) {
          const int j = j0 + W::load_col(0, fj, g);
          if (j < n) {
            const double* cp = Cb + int64_t(j) * prob.ldc;
#pragma unroll
            for (int fi = 0; fi < FI; ++fi)
#pragma unroll
              for (int cc = 0; cc < 2; ++cc) {
                const int i = i0 + W::acc_row(wi, fi, cc, tq);
                if (i < m) acc[fj][fi][cc] = cp[i];
              }
          }
        }
      }

      mbar_wait(&v_full[s], int(q / S) & 1);
      const double* Bs = V + s * P::V_ELEMS;
      if (k == P::KMAX) {
#pragma unroll
        for (int kq = 0; kq < P::KMAX / 4; ++kq) mma_kstep<W>(acc, As, Bs, wi, 0, g, kq * 4 + tq);
      } else {
        const int nq = k >> 2;
#pragma unroll 1
        for (int kq = 0; kq < nq; ++kq) mma_kstep<W>(acc, As, Bs, wi, 0, g, kq * 4 + tq);
        // scalar tail keeps the in-order FMA chain for k % 4 != 0
#pragma unroll 1
        for (int kk = nq * 4; kk < k; ++kk) {
#pragma unroll
          for (int fj = 0; fj < FJ; ++fj) {
            const double bv = Bs[W::b_off(kk, W::load_col(0, fj, g))];
#pragma unroll
            for (int fi = 0; fi < FI; ++fi)
#pragma unroll
              for (int cc = 0; cc < 2; ++cc)
                acc[fj][fi][cc] =
                    fma(As[W::a_off(W::acc_row(wi, fi, cc, tq), kk)], bv, acc[fj][fi][cc]);
          }
        }
      }
      // hand the V slot back; the group's last warp out refills it with
      // chunk q + S (same parity: this group's again). acq_rel orders the
      // four warps' reads of the slot before the async-proxy refill.
      __syncwarp();
      if (PROD) {
        if (lane == 0) mbar_arrive(&v_empty[s]);
      } else if (lane == 0 && atom_add_acq_rel_cta(&v_rel[s], 1) == P::MMA_WARPS / 2 - 1) {
        v_rel[s] = 0;
        if (q + S < q_total) issue_chunk_v<P, B_T>(prob, V, v_full, q + S, chunks, units_per_item);
      }

      if (flags & 2) continue;
#pragma unroll
      for (int fj = 0; fj < FJ; ++fj) {
        const int j = j0 + W::load_col(0, fj, g);
        if (j < n) {
          double* cp = Cb + int64_t(j) * prob.ldc;
#pragma unroll
          for (int p = 0; p < FI / 2; ++p) {
            const int i = i0 + W::acc_row(wi, 2 * p, 0, tq);  // rows i .. i+3
            const double r0 = acc[fj][2 * p][0], r1 = acc[fj][2 * p + 1][0];
            const double r2 = acc[fj][2 * p][1], r3 = acc[fj][2 * p + 1][1];
            if (vec4_ok && i + 3 < m) {
              st_global_v4(cp + i, r0, r1, r2, r3);
            } else {
              if (i < m) st_global_cs(cp + i, r0);
              if (i + 1 < m) st_global_cs(cp + i + 1, r1);
              if (i + 2 < m) st_global_cs(cp + i + 2, r2);
              if (i + 3 < m) st_global_cs(cp + i + 3, r3);
            }
          }
        }
      }
    }
    // the unit's U buffer is refilled (unit lu + 2) once all eight warps are
    // past it
    __syncwarp();
    if (PROD) {
      if (lane == 0) mbar_arrive(&u_empty[b]);
    } else if (lane == 0 && atom_add_acq_rel_cta(&u_rel[b], 1) == P::MMA_WARPS - 1) {
      u_rel[b] = 0;
      if (lu + 2 < my_units) issue_panel<P>(prob, U, u_full, lu + 2, units_per_item);
    }
  }
}

template <bool B_T, bool PROD>
cudaError_t launch_one(const StridedProblem& prob, int flags, int device, int sm_count,
                       cudaStream_t stream, int64_t* grid_out) {
  using P = PanelCfg<B_T, PROD>;
  auto kern = lrb_panel_kernel<B_T, PROD>;
  // the shared-memory opt-in is per function and device (set once each)
  static bool attr_set[64] = {false};
  const bool cached = device >= 0 && device < 64 && attr_set[device];
  if (!cached) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(P::SMEM_BYTES));
    if (e != cudaSuccess) return e;
    if (device >= 0 && device < 64) attr_set[device] = true;
  }
  int64_t grid = sm_count;
  if (prob.num_tiles < grid) grid = prob.num_tiles;
  if (grid_out) *grid_out = grid;
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(P::THREADS), P::SMEM_BYTES,
                    stream, prob, flags);
}

}  // namespace

size_t panel_smem_bytes() { return PanelCfg<true, true>::SMEM_BYTES; }
int panel_threads() { return PanelCfg<true, true>::THREADS; }

cudaError_t launch_panel(int b_t, const StridedProblem& prob, int flags, int device,
                         int sm_count, cudaStream_t stream, int64_t* grid) {
  // the producer-warpgroup form by default; LRB_PANEL_PROD=0 (probe) runs
  // the self-refilling eight-warp form
  static const bool prod = [] {
    const char* e = std::getenv("LRB_PANEL_PROD");
    return !(e && e[0] == '0');
  }();
  if (prod)
    return b_t ? launch_one<true, true>(prob, flags, device, sm_count, stream, grid)
               : launch_one<false, true>(prob, flags, device, sm_count, stream, grid);
  return b_t ? launch_one<true, false>(prob, flags, device, sm_count, stream, grid)
             : launch_one<false, false>(prob, flags, device, sm_count, stream, grid);
}

}  // namespace lrb
