// lrb_varn.cu — one persistent launch for a whole variable-size pointer-array
// batch (BASELINE cfg4: C_i = A_i (b_i x b_i) B_i (b_i x r_i), b_i in
// {256, 512, 1024}, r_i in 8..64), replacing the per-item gemm_naive_raw calls
// over separately allocated blocks (reference blr.hpp:141-175; the oracle loop
// nest dense.hpp:43-56).
//
// The per-variant bucket launches (lrb_gemm.cuh, one kernel per 8-column width
// class) pad every r_i up to its class width — 9 % of cfg4's DMMA work is
// padding — and run one launch per class, each with its own tail. This kernel
// serves every tile of every item from a single tile list:
//   * A CTA tile is 128 rows x up to 64 columns of C (4 computing warps of 32
//     rows each, all columns) fed by a producer warp through a 2-slot TMA ring
//     of 32-deep k chunks (per-item 2-D tensor maps; the B box is only as wide
//     as the item's columns, rounded to 8).
//   * The column count is a run-time property of the tile: the warps run
//     F = ceil(cols / 8) DMMA fragment columns (a compile-time specialisation
//     per F, dispatched per tile; the last fragment zero-padded), k in
//     ascending order — each C entry is one in-order FMA chain, bitwise the
//     reference's FMA-contracted loop. (Two scalar-DFMA forms of the last
//     cols % 8 columns were measured and dropped; carrying
//     them as a run-time option also cost the hot loop register spills.)
//   * Tiles are claimed dynamically (one atomic ticket per tile, taken by the
//     producer and passed to the computing warps through the ring slot), in a
//     host-chosen order that interleaves FP64-bound and HBM-bound tiles so the
//     two CTAs of an SM overlap the tensor pipe with the HBM stream, largest
//     first so the last tickets are short. The ticket counter resets itself at
//     the end of the launch (last CTA out), so graph replays need no memset.
#include <cstdint>

#include "lrb_gemm.cuh"
#include "lrb_varn.h"

namespace lrb {

// Tile configuration for F fragment columns; pitches are fixed (independent
// of F) so every specialisation reads the same shared-memory layout.
template <bool AT, bool BT, int F>
struct VarnCfg {
  static constexpr int WARPS_I = 4, WARPS_J = 1, WI = 32, WJ = 8 * F;
  static constexpr int KB = kVarnKB, MB = kVarnMB, NB = WJ;
  static constexpr int FI = WI / 8, FJ = F;
  static constexpr bool A_T = AT, B_T = BT;
  static constexpr int PMA = MB + kPad;        // A K-rows  (op(A)=N): As[kk][i]
  static constexpr int PKA = KB + kPad;        // A K-contig (op(A)=T): As[i][kk]
  static constexpr int PNB = kVarnNB + kPad;   // B K-rows  (op(B)=T): Bs[kk][j]
  static constexpr int PKB = KB + kPad;        // B K-contig (op(B)=N): Bs[j][kk]
  static constexpr bool PAIR_I = !A_T && (FI % 2 == 0);
  static constexpr bool PAIR_J = B_T && (FJ % 2 == 0);
  __device__ __forceinline__ static int load_row(int wi, int fi, int g) {
    return PAIR_I ? wi * WI + 16 * (fi >> 1) + 2 * g + (fi & 1) : wi * WI + 8 * fi + g;
  }
  __device__ __forceinline__ static int load_col(int wj, int fj, int g) {
    return PAIR_J ? wj * WJ + 16 * (fj >> 1) + 2 * g + (fj & 1) : wj * WJ + 8 * fj + g;
  }
  __device__ __forceinline__ static int acc_row(int wi, int fi, int c, int tq) {
    return PAIR_I ? wi * WI + 16 * (fi >> 1) + 2 * (2 * tq + c) + (fi & 1)
                  : wi * WI + 8 * fi + 2 * tq + c;
  }
  __device__ __forceinline__ static int a_off(int i, int kk) {
    return A_T ? i * PKA + kk : kk * PMA + i;
  }
  __device__ __forceinline__ static int b_off(int kk, int j) {
    return B_T ? kk * PNB + j : j * PKB + kk;
  }
};

template <bool AT, bool BT>
struct VarnLayout {
  static constexpr int KB = kVarnKB, MB = kVarnMB, NBMAX = kVarnNB;
  static constexpr int A_BOX = AT ? (KB + kPad) * MB : (MB + kPad) * KB;
  static constexpr int B_ELEMS_MAX = BT ? (NBMAX + kPad) * KB : (KB + kPad) * NBMAX;
  static constexpr int A_ELEMS = round_up_c(A_BOX, 16);
  static constexpr int STAGE_ELEMS = A_ELEMS + round_up_c(B_ELEMS_MAX, 16);
  static constexpr int STAGES = kVarnStages;
  static constexpr int WARPS = 4;
  // + a producer warpgroup (one active lane) that hands its registers to the
  // computing warpgroup (setmaxnreg): 64 x 32 accumulators need ~200
  static constexpr int THREADS = WARPS * 32 + 128;
  static constexpr int PROD_REGS = 48, MMA_REGS = 208;
  // stages, full + empty barriers, the slot -> tile ticket table
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * STAGE_ELEMS * 8 + size_t(STAGES) * 8 * 2 + size_t(STAGES) * 8;
  // bytes one chunk of an item with n columns lands (what expect_tx waits for)
  __device__ __forceinline__ static uint32_t chunk_bytes(int n) {
    const int bw = BT ? (NBMAX + kPad) * KB : (KB + kPad) * varn_box_cols(n);
    return uint32_t(A_BOX + bw) * 8u;
  }
};

// 64-byte descriptor load
__device__ __forceinline__ ItemDesc load_desc(const ItemDesc* p) { return *p; }

template <bool AT, bool BT, int F>
__device__ __forceinline__ void varn_tile(const ItemDesc& d, int i0, int j0,
                                          const double* smem, uint64_t* full, uint64_t* empty,
                                          int& stage, uint32_t& phase, int beta_one, int flags) {
  using Cfg = VarnCfg<AT, BT, F>;
  using L = VarnLayout<AT, BT>;
  constexpr int FI = Cfg::FI, FJ = Cfg::FJ, KB = L::KB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wi = warp, wj = 0, g = lane >> 2, tq = lane & 3;
  double acc[FJ][FI][2];
#pragma unroll
  for (int fj = 0; fj < FJ; ++fj)
#pragma unroll
    for (int fi = 0; fi < FI; ++fi) acc[fj][fi][0] = acc[fj][fi][1] = 0.0;
  if (beta_one) {
#pragma unroll
    for (int fj = 0; fj < FJ; ++fj) {
      const int j = j0 + Cfg::load_col(wj, fj, g);
      if (j < d.n) {
        const double* cp = d.C + int64_t(j) * d.ldc;
#pragma unroll
        for (int fi = 0; fi < FI; ++fi)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int i = i0 + Cfg::acc_row(wi, fi, c, tq);
            if (i < d.m) acc[fj][fi][c] = cp[i];
          }
      }
    }
  }
  bool first = true;
#pragma unroll 1
  for (int k0 = 0; k0 < d.k; k0 += KB) {
    const int kvalid = min(KB, d.k - k0);
    if (!first) mbar_wait(&full[stage], phase);  // the tile's first chunk was waited for
    first = false;
    const double* As = smem + size_t(stage) * L::STAGE_ELEMS;
    const double* Bs = As + L::A_ELEMS;
    if (kvalid == KB) {
#pragma unroll
      for (int kq = 0; kq < KB / 4; ++kq) mma_kstep<Cfg>(acc, As, Bs, wi, wj, g, kq * 4 + tq);
    } else {
      const int nq = kvalid >> 2;
#pragma unroll 1
      for (int kq = 0; kq < nq; ++kq) mma_kstep<Cfg>(acc, As, Bs, wi, wj, g, kq * 4 + tq);
#pragma unroll 1
      for (int kk = nq * 4; kk < kvalid; ++kk) {
#pragma unroll
        for (int fj = 0; fj < FJ; ++fj) {
          const double bv = Bs[Cfg::b_off(kk, Cfg::load_col(wj, fj, g))];
#pragma unroll
          for (int fi = 0; fi < FI; ++fi)
#pragma unroll
            for (int c = 0; c < 2; ++c)
              acc[fj][fi][c] = fma(As[Cfg::a_off(Cfg::acc_row(wi, fi, c, tq), kk)], bv,
                                   acc[fj][fi][c]);
        }
      }
    }
    // hand the slot back to the producer
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == L::STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (flags & 2) return;  // debug probe: no stores
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(d.C) & 15) == 0) && ((d.ldc & 1) == 0);
  const bool vec4_ok = ((reinterpret_cast<uintptr_t>(d.C) & 31) == 0) && ((d.ldc & 3) == 0);
#pragma unroll
  for (int fj = 0; fj < FJ; ++fj) {
    const int j = j0 + Cfg::load_col(wj, fj, g);
    if (j < d.n) {
      double* cp = d.C + int64_t(j) * d.ldc;
      if constexpr (Cfg::PAIR_I) {
#pragma unroll
        for (int p = 0; p < FI / 2; ++p) {
          const int i = i0 + Cfg::acc_row(wi, 2 * p, 0, tq);  // rows i .. i+3
          const double r0 = acc[fj][2 * p][0], r1 = acc[fj][2 * p + 1][0];
          const double r2 = acc[fj][2 * p][1], r3 = acc[fj][2 * p + 1][1];
          if (vec4_ok && i + 3 < d.m) {
            st_global_v4(cp + i, r0, r1, r2, r3);
          } else {
            if (i < d.m) st_global_cs(cp + i, r0);
            if (i + 1 < d.m) st_global_cs(cp + i + 1, r1);
            if (i + 2 < d.m) st_global_cs(cp + i + 2, r2);
            if (i + 3 < d.m) st_global_cs(cp + i + 3, r3);
          }
        }
      } else {
#pragma unroll
        for (int fi = 0; fi < FI; ++fi) {
          const int i = i0 + Cfg::acc_row(wi, fi, 0, tq);  // rows i, i+1
          if (vec_ok && i + 1 < d.m) {
            st_global_v2(cp + i, acc[fj][fi][0], acc[fj][fi][1]);
          } else {
            if (i < d.m) st_global_cs(cp + i, acc[fj][fi][0]);
            if (i + 1 < d.m) st_global_cs(cp + i + 1, acc[fj][fi][1]);
          }
        }
      }
    }
  }
}

template <bool AT, bool BT>
__global__ void __launch_bounds__(VarnLayout<AT, BT>::THREADS, 2)
    lrb_varn_kernel(const __grid_constant__ VarnProblem prob, const int flags) {
  using L = VarnLayout<AT, BT>;
  pdl_entry();
  const int beta_one = flags & 1;
  extern __shared__ __align__(1024) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(L::STAGES) * L::STAGE_ELEMS);
  uint64_t* empty = full + L::STAGES;
  volatile long long* slot_tile = reinterpret_cast<volatile long long*>(empty + L::STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], L::WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= L::WARPS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(L::PROD_REGS));
    // the producer: claim a tile, stream its k chunks into the ring, repeat;
    // the slot's ticket tells the computing warps which tile the chunk is of
    if (warp == L::WARPS && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t q = 0;
      // host-built tile list, or (device-built plans) the tile prefix over
      // the ordered items, searched forward from this CTA's last position
      const long long limit = prob.tiles ? prob.num_tiles : static_cast<long long>(*prob.total);
      // device-built plans: the planning kernels expanded the tile list when
      // it fit (dev_tiles, dev_cap); otherwise the prefix is searched
      const uint64_t* tiles = prob.tiles ? prob.tiles
                                         : (limit <= prob.dev_cap ? prob.dev_tiles : nullptr);
      const bool dev = tiles == nullptr;
      const int64_t count = dev ? int64_t(*prob.count) : 0;
      int64_t cursor = 0;
      // claim a ticket and decode it into (entry, m, n, k); entry -1 = done
      struct Claim {
        long long e;
        int m, n, k;
      };
      auto claim = [&]() -> Claim {
        const long long t = static_cast<long long>(atomicAdd(prob.next, 1ull));
        if (t >= limit) return Claim{-1, 0, 0, 0};
        uint64_t e;
        if (!dev) {
          e = tiles[t];
          const ItemDesc* d = prob.items + uint32_t(e >> 32);
          return Claim{static_cast<long long>(e), d->m, d->n, d->k};
        }
        const int64_t p = prefix_search(prob.prefix, count, t, &cursor);
        const uint32_t it = prob.order[p];
        const ItemDesc* d = prob.items + it;
        const int m = d->m, n = d->n, k = d->k;
        const int64_t local = t - prob.prefix[p];
        const int64_t tiles_i = (m + L::MB - 1) / L::MB;
        e = (uint64_t(it) << 32) | (uint64_t(local % tiles_i) << 16) | uint64_t(local / tiles_i);
        return Claim{static_cast<long long>(e), m, n, k};
      };
      Claim cur = claim();
#pragma unroll 1
      while (true) {
        if (q >= L::STAGES) mbar_wait(&empty[stage], phase ^ 1);
        if (cur.e < 0) {
          slot_tile[stage] = -1;  // end of the sequence
          mbar_arrive(&full[stage]);
          break;
        }
        const uint64_t e = static_cast<uint64_t>(cur.e);
        const uint32_t item = uint32_t(e >> 32);
        const int i0 = int((e >> 16) & 0xFFFF) * L::MB;
        const int j0 = int(e & 0xFFFF) * L::NBMAX;
        const void* mA = &prob.maps[2 * size_t(item)];
        const void* mB = &prob.maps[2 * size_t(item) + 1];
        if (!prob.tiles && !(flags & 16)) {  // (bit 4: probe without the fences)
          // maps written by the planning kernels (tensormap.replace): order
          // those generic-proxy writes before the TMA reads them
          fence_tensormap_acquire(mA);
          fence_tensormap_acquire(mB);
        }
        // A is single-use unless other column tiles re-read it; B is re-read
        // by every row tile of the item
        const uint64_t pol_a = cur.n <= L::NBMAX ? policy_evict_normal() : policy_evict_last();
        const uint64_t pol_b = cur.m <= L::MB ? policy_evict_normal() : policy_evict_last();
        const uint32_t bytes = L::chunk_bytes(cur.n);
        const int kk = cur.k;
        // the next ticket is claimed once this tile's chunks are all issued
        // (flags bit 3, a probe: claim it while the first chunk is in flight;
        // measured ~1 % slower on cfg4, 8.65 vs 8.56 ms: a CTA then holds a
        // ticket other CTAs could already start)
        const bool ahead = (flags & 8) != 0;
        Claim nxt{-1, 0, 0, 0};
#pragma unroll 1
        for (int k0 = 0; k0 < kk; k0 += L::KB) {
          if (k0 > 0 && q >= L::STAGES) mbar_wait(&empty[stage], phase ^ 1);
          slot_tile[stage] = static_cast<long long>(e);
          fence_proxy_async_smem();
          double* As = smem + size_t(stage) * L::STAGE_ELEMS;
          double* Bs = As + L::A_ELEMS;
          mbar_arrive_expect_tx(&full[stage], bytes);
          if (AT)
            tma_load_3d(As, mA, k0, i0, 0, &full[stage], pol_a);
          else
            tma_load_3d(As, mA, i0, k0, 0, &full[stage], pol_a);
          if (BT)
            tma_load_3d(Bs, mB, j0, k0, 0, &full[stage], pol_b);
          else
            tma_load_3d(Bs, mB, k0, j0, 0, &full[stage], pol_b);
          ++q;
          if (++stage == L::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          // the next tile is claimed and decoded while this one's first
          // chunks are in flight, so its descriptor loads stay off the ring
          if (ahead && k0 == 0) nxt = claim();
        }
        cur = ahead ? nxt : claim();
      }
      // every claim of this CTA is over: the last CTA out resets the tickets
      // for the next launch (which waits for this grid before its first claim)
      __threadfence();
      const unsigned long long done = atomicAdd(prob.next + 1, 1ull);
      if (done == gridDim.x - 1) {
        prob.next[0] = 0;
        prob.next[1] = 0;
        __threadfence();
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(L::MMA_REGS));

  int stage = 0;
  uint32_t phase = 0;
#pragma unroll 1
  while (true) {
    mbar_wait(&full[stage], phase);
    const long long te = slot_tile[stage];
    if (te < 0) break;
    const uint64_t e = static_cast<uint64_t>(te);
    const ItemDesc d = load_desc(prob.items + uint32_t(e >> 32));
    const int i0 = int((e >> 16) & 0xFFFF) * L::MB;
    const int j0 = int(e & 0xFFFF) * L::NBMAX;
    // columns of this tile, rounded up to whole 8-column fragments
    const int F = (min(L::NBMAX, d.n - j0) + 7) >> 3;
    switch (F) {
      case 1: varn_tile<AT, BT, 1>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      case 2: varn_tile<AT, BT, 2>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      case 3: varn_tile<AT, BT, 3>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      case 4: varn_tile<AT, BT, 4>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      case 5: varn_tile<AT, BT, 5>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      case 6: varn_tile<AT, BT, 6>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      case 7: varn_tile<AT, BT, 7>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
      default: varn_tile<AT, BT, 8>(d, i0, j0, smem, full, empty, stage, phase, beta_one, flags); break;
    }
  }
}

template <bool AT, bool BT>
cudaError_t launch_varn_t(const VarnProblem& p, int flags, int device, int sm_count,
                          cudaStream_t stream, int64_t* grid_out) {
  using L = VarnLayout<AT, BT>;
  auto kern = lrb_varn_kernel<AT, BT>;
  static int occ_cache[64] = {0};
  int occ = (device >= 0 && device < 64) ? occ_cache[device] : 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(L::SMEM_BYTES));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, L::THREADS, L::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (device >= 0 && device < 64) occ_cache[device] = occ;
  }
  int64_t grid = int64_t(sm_count) * occ;
  // (device-built plans: the tile count is known only on the device)
  if (p.tiles && p.num_tiles < grid) grid = p.num_tiles;
  if (grid_out) *grid_out = grid;
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(kern, dim3(unsigned(grid)), dim3(L::THREADS), L::SMEM_BYTES, stream, p, flags);
}

cudaError_t launch_varn(int a_t, int b_t, const VarnProblem& p, int flags, int device,
                        int sm_count, cudaStream_t stream, int64_t* grid) {
  if (!a_t && !b_t) return launch_varn_t<false, false>(p, flags, device, sm_count, stream, grid);
  if (!a_t && b_t) return launch_varn_t<false, true>(p, flags, device, sm_count, stream, grid);
  if (a_t && !b_t) return launch_varn_t<true, false>(p, flags, device, sm_count, stream, grid);
  return launch_varn_t<true, true>(p, flags, device, sm_count, stream, grid);
}

}  // namespace lrb
