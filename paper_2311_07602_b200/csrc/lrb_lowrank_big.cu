// lrb_lowrank_big.cu — the paper's low-rank product at rank 128 in ONE launch.
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

constexpr int kBigR = 128;            // the rank this kernel serves
constexpr int kBigKB1 = 16;           // phase-1 k chunk (b direction)
constexpr int kBigKB2 = 32;           // phase-2/3 k chunk (r direction)
constexpr int kBigP = kBigR + kPad;   // 132: pitch of T / E and the r-wide boxes
constexpr int kBigBU = kBigP * kBigKB1;            // B_U chunk  [kk][n]   2112
constexpr int kBigAV = kBigR * (kBigKB1 + kPad);   // A_Vt chunk [m][kk]   2560
constexpr int kBigAX = kBigR * (kBigKB2 + kPad);   // A_X chunk  [x][kk]   4608
constexpr int kBigBX = kBigP * kBigKB2;            // B_X chunk  [kk][y]   4224
constexpr int kBigSlot = kBigBU + kBigAV;          // 4672 doubles, 37 KB
constexpr int kBigSlots = 5;                       // 0, 1 dedicated; 2..4 inside T
constexpr int kBigT = kBigR * kBigP;               // 16896 doubles, 135 KB
constexpr int kBigTOff = 2 * kBigSlot;             // T region = slot 2's start
constexpr int kBigElems = kBigTOff + kBigT;        // 26240 doubles
constexpr int kBigMmaWarps = 8;
constexpr int kBigThreads = kBigMmaWarps * 32 + 128;
constexpr int kBigMmaRegs = 232, kBigProdRegs = 40;
constexpr size_t kBigSmem = size_t(kBigElems) * 8 + size_t(2 * kBigSlots + 1) * 8;
static_assert(kBigSlot % 16 == 0 && kBigBU % 16 == 0, "128-byte aligned TMA destinations");
static_assert(kBigAX <= kBigSlot && kBigBX <= kBigSlot, "phase-2/3 chunks fit a slot");
static_assert(kBigSlots * kBigSlot <= kBigTOff + kBigT, "slots 2..4 lie inside T");
static_assert(kBigSmem <= 232448, "shared memory per CTA");

// One phase's operand view, in the GemmCfg vocabulary mma_kstep reads: the
// kernel computes C^T = op(B)^T op(A)^T of a row-major product, so "i" is
// the row-major result's column index and "j" its row index. A' is K-rows
// (As[kk][i], pitch PA), B' is K-contiguous (Bs[j][kk], pitch PB).
template <int PA, int PB>
struct BigCfg {
  static constexpr int WI = 64, WJ = 32, FI = WI / 8, FJ = WJ / 8;
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
using Ph1 = BigCfg<kBigP, kBigKB1 + kPad>;  // A' = B_U chunk, B' = A_Vt chunk
using Ph2 = BigCfg<kBigP, kBigKB2 + kPad>;  // A' = T,         B' = A_X chunk
using Ph3 = BigCfg<kBigP, kBigP>;           // A' = B_X chunk, B' = E

struct BigProblem {
  CUtensorMap tmBU;  // (r, b, batch) view of B_U, box (132, 16, 1)
  CUtensorMap tmAV;  // (b, r, batch) view of A_Vt, box (20, 128, 1)
  CUtensorMap tmAX;  // (r, r, batch) view of A_X, box (36, 128, 1)
  CUtensorMap tmBX;  // (r, r, batch) view of B_X, box (132, 32, 1)
  double* g;
  int64_t batch;
  int block;
  int g_vec;  // G alignment: 2 = 32-byte, 1 = 16-byte, 0 = 8-byte stores
};

using Acc = double[Ph1::FJ][Ph1::FI][2];

__device__ __forceinline__ void zero_acc(Acc& acc) {
#pragma unroll
  for (int fj = 0; fj < Ph1::FJ; ++fj)
#pragma unroll
    for (int fi = 0; fi < Ph1::FI; ++fi) acc[fj][fi][0] = acc[fj][fi][1] = 0.0;
}

// the warp's accumulators into T / E (row-major [j][i], pitch 132)
__device__ __forceinline__ void stash(double* t, const Acc& acc, int wi, int wj, int g, int tq) {
#pragma unroll
  for (int fj = 0; fj < Ph1::FJ; ++fj) {
    const int j = Ph1::load_col(wj, fj, g);
#pragma unroll
    for (int p = 0; p < Ph1::FI / 2; ++p) {
      const int i = Ph1::acc_row(wi, 2 * p, 0, tq);  // i .. i+3
      sts128(t + j * kBigP + i, acc[fj][2 * p][0], acc[fj][2 * p + 1][0]);
      sts128(t + j * kBigP + i + 2, acc[fj][2 * p][1], acc[fj][2 * p + 1][1]);
    }
  }
}

__global__ void __launch_bounds__(kBigThreads, 1)
    lrb_lowrank_r128_kernel(const __grid_constant__ BigProblem p) {
  pdl_entry();
  extern __shared__ __align__(1024) double smem[];
  uint64_t* const full = reinterpret_cast<uint64_t*>(smem + kBigElems);
  uint64_t* const empty = full + kBigSlots;
  uint64_t* const t_free = empty + kBigSlots;
  double* const T = smem + kBigTOff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk1 = p.block / kBigKB1;
  constexpr int nk2 = kBigR / kBigKB2;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kBigSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBigMmaWarps);
    }
    mbar_init(t_free, kBigMmaWarps);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= kBigMmaWarps) {
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
        return smem + s * kBigSlot;
      };
#pragma unroll 1
      for (int64_t item = blockIdx.x; item < p.batch; item += gridDim.x, ++n) {
        const int z = int(item);
        int s = 0;
#pragma unroll 1
        for (int j = 0; j < nk1; ++j) {
          // slots 2..4 hold the previous item's T / E until its phase 3 ends
          if (s == 2 && j == 2 && n > 0) mbar_wait(t_free, uint32_t(n - 1) & 1);
          double* d = issue(s, uint32_t(kBigSlot) * 8u);
          tma_load_3d(d, &p.tmBU, 0, j * kBigKB1, z, &full[s], pol);
          tma_load_3d(d + kBigBU, &p.tmAV, j * kBigKB1, 0, z, &full[s], pol);
          if (++s == kBigSlots) s = 0;
        }
#pragma unroll 1
        for (int c = 0; c < nk2; ++c) {
          double* d = issue(c & 1, uint32_t(kBigAX) * 8u);
          tma_load_3d(d, &p.tmAX, c * kBigKB2, 0, z, &full[c & 1], pol);
        }
#pragma unroll 1
        for (int c = 0; c < nk2; ++c) {
          double* d = issue(c & 1, uint32_t(kBigBX) * 8u);
          tma_load_3d(d, &p.tmBX, 0, c * kBigKB2, z, &full[c & 1], pol);
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kBigMmaRegs));

  const int wi = warp & 1, wj = warp >> 1;  // 64-wide i block, 32-wide j block
  const int g = lane >> 2, tq = lane & 3;
  uint32_t fpar = 0;  // per-slot parity of the full barriers
  auto take = [&](int s) -> const double* {
    mbar_wait(&full[s], (fpar >> s) & 1);
    fpar ^= 1u << s;
    return smem + s * kBigSlot;
  };
  auto give = [&](int s) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  };
  Acc acc;
#pragma unroll 1
  for (int64_t item = blockIdx.x; item < p.batch; item += gridDim.x) {
    // phase 1: T^T = B_U^T A_Vt^T, k = 0 .. b-1 ascending
    zero_acc(acc);
    int s = 0;
#pragma unroll 1
    for (int j = 0; j < nk1; ++j) {
      const double* d = take(s);
#pragma unroll
      for (int kq = 0; kq < kBigKB1 / 4; ++kq)
        mma_kstep<Ph1>(acc, d, d + kBigBU, wi, wj, g, kq * 4 + tq);
      give(s);
      if (++s == kBigSlots) s = 0;
    }
    // every warp is past the phase-1 slots that T overlays
    named_barrier_sync(1, kBigMmaWarps * 32);
    stash(T, acc, wi, wj, g, tq);
    named_barrier_sync(1, kBigMmaWarps * 32);
    // phase 2: E^T = T^T A_X^T, m = 0 .. r-1 ascending
    zero_acc(acc);
#pragma unroll 1
    for (int c = 0; c < nk2; ++c) {
      const double* d = take(c & 1);
#pragma unroll
      for (int kq = 0; kq < kBigKB2 / 4; ++kq)
        mma_kstep<Ph2>(acc, T + c * kBigKB2 * kBigP, d, wi, wj, g, kq * 4 + tq);
      give(c & 1);
    }
    named_barrier_sync(1, kBigMmaWarps * 32);
    stash(T, acc, wi, wj, g, tq);  // E replaces T
    named_barrier_sync(1, kBigMmaWarps * 32);
    // phase 3: G^T = B_X^T E^T, n = 0 .. r-1 ascending
    zero_acc(acc);
#pragma unroll 1
    for (int c = 0; c < nk2; ++c) {
      const double* d = take(c & 1);
#pragma unroll
      for (int kq = 0; kq < kBigKB2 / 4; ++kq)
        mma_kstep<Ph3>(acc, d, T + c * kBigKB2, wi, wj, g, kq * 4 + tq);
      give(c & 1);
    }
    // E is read: the producer may land the next item's chunks over it
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(t_free);
    // G (row-major [x][y]) = C'[i = y][j = x]: four consecutive y per lane
    double* gi = p.g + item * int64_t(kBigR) * kBigR;
#pragma unroll
    for (int fj = 0; fj < Ph1::FJ; ++fj) {
      const int x = Ph1::load_col(wj, fj, g);
#pragma unroll
      for (int q = 0; q < Ph1::FI / 2; ++q) {
        const int y = Ph1::acc_row(wi, 2 * q, 0, tq);
        double* o = gi + x * kBigR + y;
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

}  // namespace

// The fused rank-128 path applies: rank 128, block a multiple of 16 (>= 48,
// so the ring reaches slot 2 before T is needed), 16-byte aligned roles, and
// a batch whose item index fits the tensor map's coordinate.
bool lowrank_big_eligible(int64_t batch, int64_t block, int64_t rank, const void* a_vt,
                          const void* b_u, const void* a_x, const void* b_x) {
  const char* e = std::getenv("LRB_LOWRANK_FUSED_BIG");
  if (e && e[0] == '0') return false;
  const uintptr_t al = reinterpret_cast<uintptr_t>(a_vt) | reinterpret_cast<uintptr_t>(b_u) |
                       reinterpret_cast<uintptr_t>(a_x) | reinterpret_cast<uintptr_t>(b_x);
  return rank == kBigR && block % kBigKB1 == 0 && block >= 3 * kBigKB1 && block <= INT32_MAX &&
         (al & 15) == 0 && batch <= INT32_MAX && encode_fn() != nullptr;
}

lrb_status run_lowrank_big(lrb_ctx* ctx, int64_t batch, int64_t block, const double* a_vt,
                           const double* b_u, const double* a_x, const double* b_x, double* g,
                           cudaStream_t s) {
  BigProblem p;
  std::memset(&p, 0, sizeof(p));
  const int64_t r = kBigR;
  const bool ok = encode_big(&p.tmBU, b_u, r, block, batch, kBigP, kBigKB1) &&
                  encode_big(&p.tmAV, a_vt, block, r, batch, kBigKB1 + kPad, kBigR) &&
                  encode_big(&p.tmAX, a_x, r, r, batch, kBigKB2 + kPad, kBigR) &&
                  encode_big(&p.tmBX, b_x, r, r, batch, kBigP, kBigKB2);
  if (!ok) return fail(ctx, LRB_ERR_CUDA, "lrb_lowrank_multiply: tensor map encoding failed");
  p.g = g;
  p.batch = batch;
  p.block = int(block);
  const uintptr_t ga = reinterpret_cast<uintptr_t>(g);
  p.g_vec = (ga & 31) == 0 ? 2 : (ga & 15) == 0 ? 1 : 0;
  static bool attr_set[64] = {false};
  const int dev = ctx->device;
  if (!(dev >= 0 && dev < 64 && attr_set[dev])) {
    LRB_CUDA_TRY(ctx, cudaFuncSetAttribute(lrb_lowrank_r128_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kBigSmem)));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const int64_t grid = std::min<int64_t>(batch, ctx->sm_count);
  if (grid <= 0) return LRB_OK;
  LRB_CUDA_TRY(ctx, launch_pdl(lrb_lowrank_r128_kernel, dim3(unsigned(grid)), dim3(kBigThreads),
                                kBigSmem, s, p));
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  return LRB_OK;
}

}  // namespace lrb
