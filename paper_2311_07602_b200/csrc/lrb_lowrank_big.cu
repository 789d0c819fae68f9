// lrb_lowrank_big.cu — the paper's low-rank product at ranks 64, 96 and 128 in
// ONE launch (the geometry below is described at rank 128).
//
//   G_i = A_X_i (A_Vt_i B_U_i) B_X_i        (arXiv 2311.07602, Algorithm 1)
//
// over a LowRankBatch (every role row-major and packed, reference
// low_rank.hpp:109-176; drivers fused_multiply / packed_multiply,
// kernels.hpp:131-349; oracle low_rank_multiply_reference_raw,
// low_rank.hpp:73-87).
//
// Why. At r > 32 the product ran as three batched GEMMs with T = A_Vt B_U and
// E = A_X T in a workspace: at r = 128 every item then writes and re-reads
// 4 r^2 doubles of intermediates (0.5 MB of its 2.5 MB), and the 128 x 64
// tiles of the first GEMM read A_Vt twice — DRAM 1.26x the algorithmic bytes
// (profiles/traffic.json, lr_r128_b1024). Here one CTA owns an item at a
// time and keeps T and E on chip, so the operands leave DRAM once and G is
// written once:
//   * Eight MMA warps (two warpgroups; warp tile 64 x 32 of the 128 x 128
//     output, 64 accumulators) and a producer warpgroup whose first lane
//     issues every TMA load; setmaxnreg moves the producer's registers to the
//     MMA warps (40 / 232 per thread, the panel kernel's split).
//   * Phase 1, T = A_Vt B_U (K = b): 16-deep k chunks of B_U (16 x 128, pitch
//     132) and A_Vt (128 x 16, pitch 20) through a ring of five 37 KB slots.
//     Phase 2, E = A_X T (K = r): T in shared memory (128 x 128, pitch 132),
//     A_X in 32-column chunks. Phase 3, G = E B_X (K = r): E in place of T,
//     B_X in 32-row chunks. G leaves in 32-byte streaming stores.
//   * T (135 KB) shares its memory with ring slots 2..4, which only phase 1
//     uses: the producer issues the next item's chunks into slots 0 and 1 as
//     soon as they are free and into slots 2..4 once every MMA warp is past
//     phase 3 (the t_free barrier), so the ring keeps running across items.
// Each product is an in-order FMA chain over its inner index (DMMA 8x8x4
// k-steps in ascending k), so G is bitwise the three-GEMM path's and the
// oracle's FMA-chain result.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "lrb_gemm.cuh"
#include "lrb_internal.h"

namespace lrb {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn();  // lrb_api.cu

namespace {

// Geometry per rank R. Ranks 96 and 128: eight MMA warps in a 2 x 4 grid (an
// R/2 x R/4 warp tile each) plus a producer warpgroup that hands its registers
// over, one CTA per SM. Rank 64: four MMA warps in a 2 x 2 grid (32 x 32 warp
// tiles) plus one producer warp, TWO CTAs per SM — its phases are short
// (64-deep inner products between CTA barriers), so a second CTA keeps the
// DMMA pipe busy while the first stashes T / E or stores G.
template <int R>
struct Big {
  static constexpr int MMA_WARPS = R == 64 ? 4 : 8;
  static constexpr int WARPS_J = MMA_WARPS / 2;
  static constexpr int CTAS = R == 64 ? 2 : 1;
  static constexpr bool HANDOVER = R != 64;      // setmaxnreg producer -> MMA warps
  static constexpr int THREADS = MMA_WARPS * 32 + (HANDOVER ? 128 : 32);
  static constexpr int KB1 = 16;                 // phase-1 k chunk (b direction)
  static constexpr int KB2 = 32;                 // phase-2/3 k chunk (r direction)
  static constexpr int P = R + kPad;             // pitch of T / E and the r-wide boxes
  static constexpr int BU = P * KB1;             // B_U chunk  [kk][n]
  static constexpr int AV = R * (KB1 + kPad);    // A_Vt chunk [m][kk]
  static constexpr int AX = R * (KB2 + kPad);    // A_X chunk  [x][kk]
  static constexpr int BX = P * KB2;             // B_X chunk  [kk][y]
  static constexpr int SLOT = BU + AV;           // R = 128: 4672 doubles, 37 KB
  static constexpr int SLOTS = 5;                // 0, 1 dedicated; 2..4 share memory with T
  static constexpr int T = R * P;                // R = 128: 16896 doubles, 135 KB
  static constexpr int TOFF = 2 * SLOT;          // T region = slot 2's start
  static constexpr int ELEMS = TOFF + (T > 3 * SLOT ? T : 3 * SLOT);
  static constexpr size_t SMEM = size_t(ELEMS) * 8 + size_t(2 * SLOTS + 1) * 8;
  static_assert(SLOT % 16 == 0 && BU % 16 == 0, "128-byte aligned TMA destinations");
  static_assert(AX <= SLOT && BX <= SLOT, "phase-2/3 chunks fit a slot");
  static_assert(R % KB2 == 0 && R % 32 == 0, "whole chunks, 16-row paired fragments");
  static_assert(SMEM * CTAS + 1024 * CTAS <= 233472, "shared memory per SM");
};
constexpr int kBigMmaRegs = 232, kBigProdRegs = 40;

// One phase's operand view, in the GemmCfg vocabulary mma_kstep reads: the
// kernel computes C^T = op(B)^T op(A)^T of a row-major product, so "i" is
// the row-major result's column index and "j" its row index. A' is K-rows
// (As[kk][i], pitch PA), B' is K-contiguous (Bs[j][kk], pitch PB).
template <int R, int PA, int PB>
struct BigCfg {
  static constexpr int WI = R / 2, WJ = R / Big<R>::WARPS_J, FI = WI / 8, FJ = WJ / 8;
  static constexpr bool PAIR_I = true, PAIR_J = false;
  __device__ __forceinline__ static int load_row(int wi, int fi, int g) {
    return wi * WI + 16 * (fi >> 1) + 2 * g + (fi & 1);
  }
  __device__ __forceinline__ static int load_col(int wj, int fj, int g) { return wj * WJ + 8 * fj + g; }
  __device__ __forceinline__ static int acc_row(int wi, int fi, int c, int tq) {
    return wi * WI + 16 * (fi >> 1) + 2 * (2 * tq + c) + (fi & 1);
  }
  __device__ __forceinline__ static int a_off(int i, int kk) { return kk * PA + i; }
  __device__ __forceinline__ static int b_off(int kk, int j) { return j * PB + kk; }
};

struct BigProblem {
  CUtensorMap tmBU;  // (r, b, batch) view of B_U, box (r + 4, KB1, 1)
  CUtensorMap tmAV;  // (b, r, batch) view of A_Vt, box (KB1 + 4, r, 1)
  CUtensorMap tmAX;  // (r, r, batch) view of A_X, box (36, r, 1)
  CUtensorMap tmBX;  // (r, r, batch) view of B_X, box (r + 4, 32, 1)
  double* g;
  int64_t batch;
  int block;
  int g_vec;  // G alignment: 2 = 32-byte, 1 = 16-byte, 0 = 8-byte stores
};

template <class Cfg>
__device__ __forceinline__ void zero_acc(double (&acc)[Cfg::FJ][Cfg::FI][2]) {
#pragma unroll
  for (int fj = 0; fj < Cfg::FJ; ++fj)
#pragma unroll
    for (int fi = 0; fi < Cfg::FI; ++fi) acc[fj][fi][0] = acc[fj][fi][1] = 0.0;
}

// the warp's accumulators into T / E (row-major [j][i], pitch P)
template <class Cfg, int P>
__device__ __forceinline__ void stash(double* t, const double (&acc)[Cfg::FJ][Cfg::FI][2], int wi,
                                      int wj, int g, int tq) {
#pragma unroll
  for (int fj = 0; fj < Cfg::FJ; ++fj) {
    const int j = Cfg::load_col(wj, fj, g);
#pragma unroll
    for (int p = 0; p < Cfg::FI / 2; ++p) {
      const int i = Cfg::acc_row(wi, 2 * p, 0, tq);  // i .. i+3
      sts128(t + j * P + i, acc[fj][2 * p][0], acc[fj][2 * p + 1][0]);
      sts128(t + j * P + i + 2, acc[fj][2 * p][1], acc[fj][2 * p + 1][1]);
    }
  }
}

template <int R>
__global__ void __launch_bounds__(Big<R>::THREADS, Big<R>::CTAS)
    lrb_lowrank_big_kernel(const __grid_constant__ BigProblem p) {
  using K = Big<R>;
  constexpr int kBigMmaWarps = K::MMA_WARPS;
  using Ph1 = BigCfg<R, K::P, K::KB1 + kPad>;  // A' = B_U chunk, B' = A_Vt chunk
  using Ph2 = BigCfg<R, K::P, K::KB2 + kPad>;  // A' = T,         B' = A_X chunk
  using Ph3 = BigCfg<R, K::P, K::P>;           // A' = B_X chunk, B' = E
  constexpr int SLOTS = K::SLOTS;
  pdl_entry();
  extern __shared__ __align__(1024) double smem[];
  uint64_t* const full = reinterpret_cast<uint64_t*>(smem + K::ELEMS);
  uint64_t* const empty = full + SLOTS;
  uint64_t* const t_free = empty + SLOTS;
  double* const T = smem + K::TOFF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk1 = p.block / K::KB1;
  constexpr int nk2 = R / K::KB2;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBigMmaWarps);
    }
    mbar_init(t_free, kBigMmaWarps);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= kBigMmaWarps) {
    if constexpr (K::HANDOVER)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kBigProdRegs));
    if (warp == kBigMmaWarps && lane == 0) {
      // producer: per item, the phase-1 chunks round-robin over the five
      // slots, then the A_X and B_X chunks over slots 0 / 1
      uint32_t epar = 0;  // per-slot parity of the empty barriers
      // operands are read once; the k-contiguous A_Vt / A_X boxes read 4 pad
      // columns of the next chunk, which must still be in L2 when it lands
      const uint64_t pol = policy_evict_normal();
      int64_t n = 0;
      auto issue = [&](int s, uint32_t bytes) -> double* {
        mbar_wait(&empty[s], ((epar >> s) & 1) ^ 1);
        epar ^= 1u << s;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[s], bytes);
        return smem + s * K::SLOT;
      };
#pragma unroll 1
      for (int64_t item = blockIdx.x; item < p.batch; item += gridDim.x, ++n) {
        const int z = int(item);
        int s = 0;
#pragma unroll 1
        for (int j = 0; j < nk1; ++j) {
          // slots 2..4 hold the previous item's T / E until its phase 3 ends
          if (s == 2 && j == 2 && n > 0) mbar_wait(t_free, uint32_t(n - 1) & 1);
          double* d = issue(s, uint32_t(K::SLOT) * 8u);
          tma_load_3d(d, &p.tmBU, 0, j * K::KB1, z, &full[s], pol);
          tma_load_3d(d + K::BU, &p.tmAV, j * K::KB1, 0, z, &full[s], pol);
          if (++s == SLOTS) s = 0;
        }
#pragma unroll 1
        for (int c = 0; c < nk2; ++c) {
          double* d = issue(c & 1, uint32_t(K::AX) * 8u);
          tma_load_3d(d, &p.tmAX, c * K::KB2, 0, z, &full[c & 1], pol);
        }
#pragma unroll 1
        for (int c = 0; c < nk2; ++c) {
          double* d = issue(c & 1, uint32_t(K::BX) * 8u);
          tma_load_3d(d, &p.tmBX, 0, c * K::KB2, z, &full[c & 1], pol);
        }
      }
    }
    return;
  }
  if constexpr (K::HANDOVER)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kBigMmaRegs));

  const int wi = warp & 1, wj = warp >> 1;  // R/2-wide i block, WJ-wide j block
  const int g = lane >> 2, tq = lane & 3;
  uint32_t fpar = 0;  // per-slot parity of the full barriers
  auto take = [&](int s) -> const double* {
    mbar_wait(&full[s], (fpar >> s) & 1);
    fpar ^= 1u << s;
    return smem + s * K::SLOT;
  };
  auto give = [&](int s) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  };
  double acc[Ph1::FJ][Ph1::FI][2];
#pragma unroll 1
  for (int64_t item = blockIdx.x; item < p.batch; item += gridDim.x) {
    // phase 1: T^T = B_U^T A_Vt^T, k = 0 .. b-1 ascending
    zero_acc<Ph1>(acc);
    int s = 0;
#pragma unroll 1
    for (int j = 0; j < nk1; ++j) {
      const double* d = take(s);
#pragma unroll
      for (int kq = 0; kq < K::KB1 / 4; ++kq)
        mma_kstep<Ph1>(acc, d, d + K::BU, wi, wj, g, kq * 4 + tq);
      give(s);
      if (++s == SLOTS) s = 0;
    }
    // every warp is past the phase-1 slots that T overlays
    named_barrier_sync(1, kBigMmaWarps * 32);
    stash<Ph1, K::P>(T, acc, wi, wj, g, tq);
    named_barrier_sync(1, kBigMmaWarps * 32);
    // phase 2: E^T = T^T A_X^T, m = 0 .. r-1 ascending
    zero_acc<Ph1>(acc);
#pragma unroll 1
    for (int c = 0; c < nk2; ++c) {
      const double* d = take(c & 1);
#pragma unroll
      for (int kq = 0; kq < K::KB2 / 4; ++kq)
        mma_kstep<Ph2>(acc, T + c * K::KB2 * K::P, d, wi, wj, g, kq * 4 + tq);
      give(c & 1);
    }
    named_barrier_sync(1, kBigMmaWarps * 32);
    stash<Ph1, K::P>(T, acc, wi, wj, g, tq);  // E replaces T
    named_barrier_sync(1, kBigMmaWarps * 32);
    // phase 3: G^T = B_X^T E^T, n = 0 .. r-1 ascending
    zero_acc<Ph1>(acc);
#pragma unroll 1
    for (int c = 0; c < nk2; ++c) {
      const double* d = take(c & 1);
#pragma unroll
      for (int kq = 0; kq < K::KB2 / 4; ++kq)
        mma_kstep<Ph3>(acc, d, T + c * K::KB2, wi, wj, g, kq * 4 + tq);
      give(c & 1);
    }
    // E is read: the producer may land the next item's chunks over it
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(t_free);
    // G (row-major [x][y]) = C'[i = y][j = x]: four consecutive y per lane
    double* gi = p.g + item * int64_t(R) * R;
#pragma unroll
    for (int fj = 0; fj < Ph1::FJ; ++fj) {
      const int x = Ph1::load_col(wj, fj, g);
#pragma unroll
      for (int q = 0; q < Ph1::FI / 2; ++q) {
        const int y = Ph1::acc_row(wi, 2 * q, 0, tq);
        double* o = gi + x * R + y;
        if (p.g_vec == 2) {
          st_global_v4(o, acc[fj][2 * q][0], acc[fj][2 * q + 1][0], acc[fj][2 * q][1],
                       acc[fj][2 * q + 1][1]);
        } else if (p.g_vec == 1) {
          st_global_v2(o, acc[fj][2 * q][0], acc[fj][2 * q + 1][0]);
          st_global_v2(o + 2, acc[fj][2 * q][1], acc[fj][2 * q + 1][1]);
        } else {
          st_global_cs(o, acc[fj][2 * q][0]);
          st_global_cs(o + 1, acc[fj][2 * q + 1][0]);
          st_global_cs(o + 2, acc[fj][2 * q][1]);
          st_global_cs(o + 3, acc[fj][2 * q + 1][1]);
        }
      }
    }
  }
}

bool encode_big(CUtensorMap* map, const double* base, int64_t d0, int64_t d1, int64_t batch,
                int b0, int b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(batch)};
  cuuint64_t strides[2] = {cuuint64_t(d0 * 8), cuuint64_t(d0 * d1 * 8)};
  cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(b1), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int R>
lrb_status run_big_t(lrb_ctx* ctx, int64_t batch, int64_t block, const double* a_vt,
                     const double* b_u, const double* a_x, const double* b_x, double* g,
                     cudaStream_t s) {
  using K = Big<R>;
  BigProblem p;
  std::memset(&p, 0, sizeof(p));
  const int64_t r = R;
  const bool ok = encode_big(&p.tmBU, b_u, r, block, batch, K::P, K::KB1) &&
                  encode_big(&p.tmAV, a_vt, block, r, batch, K::KB1 + kPad, R) &&
                  encode_big(&p.tmAX, a_x, r, r, batch, K::KB2 + kPad, R) &&
                  encode_big(&p.tmBX, b_x, r, r, batch, K::P, K::KB2);
  if (!ok) return fail(ctx, LRB_ERR_CUDA, "lrb_lowrank_multiply: tensor map encoding failed");
  p.g = g;
  p.batch = batch;
  p.block = int(block);
  const uintptr_t ga = reinterpret_cast<uintptr_t>(g);
  p.g_vec = (ga & 31) == 0 ? 2 : (ga & 15) == 0 ? 1 : 0;
  static bool attr_set[64] = {false};
  const int dev = ctx->device;
  if (!(dev >= 0 && dev < 64 && attr_set[dev])) {
    LRB_CUDA_TRY(ctx, cudaFuncSetAttribute(lrb_lowrank_big_kernel<R>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(K::SMEM)));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const int64_t grid = std::min<int64_t>(batch, int64_t(ctx->sm_count) * K::CTAS);
  if (grid <= 0) return LRB_OK;
  LRB_CUDA_TRY(ctx, launch_pdl(lrb_lowrank_big_kernel<R>, dim3(unsigned(grid)), dim3(K::THREADS),
                                K::SMEM, s, p));
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  return LRB_OK;
}

int big_kb1(int64_t) { return Big<128>::KB1; }

}  // namespace

// The fused path applies: rank 64, 96 or 128, block a multiple of the phase-1
// chunk (and at least three chunks, so the ring reaches slot 2 before T is
// needed), 16-byte aligned roles, and a batch whose item index fits the
// tensor map's coordinate. LRB_LOWRANK_FUSED_BIG=0 turns it off;
// LRB_LOWRANK_FUSED_BIG=128 keeps it to rank 128 (A/B probes).
bool lowrank_big_eligible(int64_t batch, int64_t block, int64_t rank, const void* a_vt,
                          const void* b_u, const void* a_x, const void* b_x) {
  const char* e = std::getenv("LRB_LOWRANK_FUSED_BIG");
  if (e && e[0] == '0') return false;
  if (!(rank == 64 || rank == 96 || rank == 128)) return false;
  if (e && e[0] && std::atoi(e) > 1 && std::atoi(e) != rank) return false;
  const uintptr_t al = reinterpret_cast<uintptr_t>(a_vt) | reinterpret_cast<uintptr_t>(b_u) |
                       reinterpret_cast<uintptr_t>(a_x) | reinterpret_cast<uintptr_t>(b_x);
  const int kb1 = big_kb1(rank);
  return block % kb1 == 0 && block >= 3 * kb1 && block <= INT32_MAX && (al & 15) == 0 &&
         batch <= INT32_MAX && encode_fn() != nullptr;
}

lrb_status run_lowrank_big(lrb_ctx* ctx, int64_t batch, int64_t block, int64_t rank,
                           const double* a_vt, const double* b_u, const double* a_x,
                           const double* b_x, double* g, cudaStream_t s) {
  if (rank == 64) return run_big_t<64>(ctx, batch, block, a_vt, b_u, a_x, b_x, g, s);
  if (rank == 96) return run_big_t<96>(ctx, batch, block, a_vt, b_u, a_x, b_x, g, s);
  return run_big_t<128>(ctx, batch, block, a_vt, b_u, a_x, b_x, g, s);
}

}  // namespace lrb
