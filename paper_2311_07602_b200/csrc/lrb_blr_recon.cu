// lrb_blr_recon.cu — the off-diagonal tiles of BlrMatrix::reconstruct_dense
// (reference blr.hpp:62-86: out tile (i, j) = dense_gemm_naive(dense_gemm_naive(
// U_ij, X_ij), Vt_ij)) as ONE write-streaming kernel.
//
// The output (n x n, 2 GiB on the bench shape) is ~90 % of the bytes, so the
// kernel is built around keeping the TMA store stream full:
//   * unit = (tile q, 64-row block, 256-column half): a producer warp lands
//     the half's Vt_ij (two 3-D boxes of 128 + 4 columns x r rows), the
//     block's U_ij rows (one box of r + 4 columns x 64 rows from the [D_i |
//     U_i*] row panel) and X_ij (one bulk copy) into a 2-slot ring;
//   * eight computing warps (a 16 x 32 quarter-strip each) form UX = U X on
//     DMMA (rounded, the reference's first product) into shared memory, then
//     each 64 x 64 block of (UX) Vt on DMMA, k ascending — both chains as the
//     reference orders them, so results are bitwise the FMA-chain oracle;
//   * each warp stages its 16 x 32 part of every 64 x 64 output block in the
//     128-byte swizzle and hands it to the TMA engine itself (two 16 x 16
//     boxes); three staging buffers per warp rotate, so the warps never meet
//     at a barrier and two sub-blocks per warp are in flight while the next
//     one is computed.
// The diagonal tiles are copied by blr_diag_kernel (lrb_blr.cu) before it.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "lrb_device.cuh"
#include "lrb_internal.h"

namespace lrb {

bool encode_operand(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                    int64_t stride, int64_t zdim, int box_in, int box_out);

namespace {

constexpr int kRPad = 4;
constexpr int kRWarps = 8;
constexpr int kRThreads = kRWarps * 32 + 32;  // + the producer warp
constexpr int kRMaxRank = 16;
constexpr int kRHalf = 256;                 // output columns per unit
constexpr int kRBox = 128;                  // Vt box columns (+ kRPad)
constexpr int kVtElems = (kRHalf / kRBox) * (kRBox + kRPad) * kRMaxRank;  // per slot
constexpr int kUElems = 64 * (kRMaxRank + kRPad);
constexpr int kXElems = kRMaxRank * kRMaxRank;
constexpr int kSlotElems = kVtElems + kUElems + kXElems;
constexpr int kStageBufs = 3;                  // per warp
constexpr int kWarpStage = 16 * 32;            // one warp's 16 x 32 output sub-block
constexpr int kUxElems = 16 * (kRMaxRank + kRPad);  // one warp's UX rows
constexpr size_t kRSmem = size_t(kRWarps) * kStageBufs * kWarpStage * 8 +
                          size_t(2) * kSlotElems * 8 + size_t(kRWarps) * kUxElems * 8 + 64;

struct ReconProblem {
  CUtensorMap tmVt;   // stacked Vt: (b, r, Q) row-major per item     box (132, r)
  CUtensorMap tmU;    // [D_i | U_i*] rows: (P, n)                  box (r + 4, 64)
  CUtensorMap tmOut;  // out: (n, n) row-major                       box (16, 16), 128B swizzle
  const double* x;    // X_q, (j, i) order
  int T, b, r, n, P;
  int rb_per_tile, halves;
  long long units;
};

__global__ void __launch_bounds__(kRThreads, 1)
    blr_recon_kernel(const __grid_constant__ ReconProblem p) {
  pdl_entry();
  extern __shared__ __align__(1024) double smem[];
  // per-warp staging first (every 2 KB box 1024-B aligned for the swizzle),
  // then the operand ring (Vt | U | X per slot), then per-warp UX rows
  double* stage = smem;
  double* ring = stage + size_t(kRWarps) * kStageBufs * kWarpStage;
  double* uxs_all = ring + 2 * size_t(kSlotElems);
  uint64_t* full = reinterpret_cast<uint64_t*>(uxs_all + size_t(kRWarps) * kUxElems);
  uint64_t* empty = full + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = p.r, rp = r + kRPad;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int Tm1 = p.T - 1;
  auto decode = [&](long long u, int* q, int* i, int* jp, int* rb, int* half) {
    const int per_tile = p.rb_per_tile * p.halves;
    *q = int(u / per_tile);
    const int w = int(u - (long long)(*q) * per_tile);
    *rb = w / p.halves;
    *half = w - *rb * p.halves;
    const int j = *q / Tm1, ip = *q - j * Tm1;
    *i = ip < j ? ip : ip + 1;
    *jp = j < *i ? j : j - 1;
  };

  if (warp == kRWarps) {  // the producer
    if (lane == 0) {
      const uint32_t bytes =
          uint32_t((kRHalf / kRBox) * (kRBox + kRPad) * r + 64 * rp + r * r) * 8u;
      const uint64_t pol = policy_evict_normal(), pol_keep = policy_evict_last();
      int slot = 0;
      uint32_t phase = 0;
      long long nq = 0;
#pragma unroll 1
      for (long long u = blockIdx.x; u < p.units; u += gridDim.x, ++nq) {
        int q, i, jp, rb, half;
        decode(u, &q, &i, &jp, &rb, &half);
        if (nq >= 2) mbar_wait(&empty[slot], phase ^ 1);
        double* vt = ring + size_t(slot) * kSlotElems;
        double* us = vt + kVtElems;
        double* xq = us + kUElems;
        mbar_arrive_expect_tx(&full[slot], bytes);
        for (int c = 0; c < kRHalf / kRBox; ++c)
          tma_load_3d(vt + c * (kRBox + kRPad) * r, &p.tmVt, half * kRHalf + c * kRBox, 0, q,
                      &full[slot], pol_keep);
        tma_load_3d(us, &p.tmU, p.b + jp * r, i * p.b + rb * 64, 0, &full[slot], pol);
        bulk_g2s(xq, p.x + int64_t(q) * r * r, uint32_t(r * r * 8), &full[slot], pol);
        if (++slot == 2) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  const int g = lane >> 2, tq = lane & 3;
  const int row0 = (warp & 3) * 16;  // this warp's 16 rows of the 64-row block
  const int colw = (warp >> 2) * 32;  // and its 32 columns of each 64-column block
  double* uxs = uxs_all + size_t(warp) * kUxElems;  // 16 x (r + 4), this warp's rows
  double* wstage = stage + size_t(warp) * kStageBufs * kWarpStage;
  int slot = 0;
  uint32_t phase = 0;
  long long nblk = 0;  // sub-blocks this warp staged (its buffer rotation)
#pragma unroll 1
  for (long long u = blockIdx.x; u < p.units; u += gridDim.x) {
    int q, i, jp, rb, half;
    decode(u, &q, &i, &jp, &rb, &half);
    mbar_wait(&full[slot], phase);
    const double* vt = ring + size_t(slot) * kSlotElems;
    const double* us = vt + kVtElems;
    const double* xq = us + kUElems;
    // this warp's UX rows = U (16 x r) X (r x r), p ascending (both warps of
    // a row band form the same rows: no cross-warp dependency)
    for (int f = 0; f < 2; ++f)
      for (int c0 = 0; c0 < r; c0 += 8) {
        double d0 = 0.0, d1 = 0.0;
        for (int k0 = 0; k0 < r; k0 += 4)
          dmma_8x8x4(d0, d1, us[(row0 + 8 * f + g) * rp + k0 + tq], xq[(k0 + tq) * r + c0 + g]);
        double* dst = uxs + (8 * f + g) * rp + c0 + 2 * tq;
        dst[0] = d0;
        dst[1] = d1;
      }
    __syncwarp();
    // four 64 x 64 output blocks of (UX) Vt, k ascending; this warp's 16 x 32
    // part of each leaves through its own two TMA stores (16 x 16 boxes).
    // Two blocks at a time: 16 independent DMMA chains per warp keep the
    // tensor pipe busy through the DMMA latency (k = r is only 4 steps deep)
#pragma unroll 1
    for (int cp = 0; cp < kRHalf / 64; cp += 2) {
      double acc[2][2][4][2];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 4; ++h) acc[e][f][h][0] = acc[e][f][h][1] = 0.0;
#pragma unroll 1
      for (int k0 = 0; k0 < r; k0 += 4) {
        double a[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) a[f] = uxs[(8 * f + g) * rp + k0 + tq];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cb = cp + e;
          const double* vb = vt + (cb / 2) * (kRBox + kRPad) * r + (cb % 2) * 64 + colw;
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
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cb = cp + e;
        // this warp's staging buffer: free once its stores of kStageBufs
        // sub-blocks ago have read it
        double* st = wstage + size_t(nblk % kStageBufs) * kWarpStage;
        if (lane == 0) bulk_wait_group_read<kStageBufs - 1>();
        __syncwarp();
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int row = 8 * f + g;  // row within the warp's 16; row % 8 == g
            const int box = h >> 1, chunk = ((h & 1) << 2) | tq;
            sts128(st + box * 256 + row * 16 + ((chunk ^ g) << 1), acc[e][f][h][0],
                   acc[e][f][h][1]);
          }
        fence_proxy_async_shared_cta();
        __syncwarp();
        if (lane == 0) {
          const int x0 = (q / Tm1) * p.b + half * kRHalf + cb * 64 + colw;
          const int y0 = i * p.b + rb * 64 + row0;
          tma_store_2d(&p.tmOut, st, x0, y0);
          tma_store_2d(&p.tmOut, st + 256, x0 + 16, y0);
          bulk_commit_group();
        }
        ++nblk;
      }
    }
    if (++slot == 2) {
      slot = 0;
      phase ^= 1;
    }
  }
  if (lane == 0) bulk_wait_group0();  // the stores land before the grid completes
}
}  // namespace

// The whole off-diagonal part of the reconstruction in one launch, or false
// (nothing launched) when the shape is outside what the kernel serves:
// r a multiple of 8 up to 16, b a multiple of 256, TMA-addressable buffers.
bool launch_blr_recon(lrb_ctx* ctx, const double* vtcol, const double* dcat, const double* x,
                      double* out, int64_t T, int64_t b, int64_t r, int64_t P, cudaStream_t s,
                      lrb_status* st) {
  const int64_t n = T * b, Q = T * (T - 1);
  if (T < 2 || r % 8 != 0 || r > kRMaxRank || b % kRHalf != 0 || Q > INT32_MAX) return false;
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    return false;
  ReconProblem p;
  std::memset(&p, 0, sizeof(p));
  // out: 2-D (n columns, n rows), box 16 x 64, 128-byte swizzle
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr) !=
            cudaSuccess ||
        qr != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return false;
    }
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  }
  {
    cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(n)};
    cuuint64_t strides[1] = {cuuint64_t(n * 8)};
    cuuint32_t box[2] = {16, 16};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&p.tmOut, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  const bool ok = encode_operand(&p.tmVt, vtcol, b, r, b, r * b, Q, kRBox + kRPad, int(r)) &&
                  encode_operand(&p.tmU, dcat, P, n, P, 0, 1, int(r) + kRPad, 64);
  if (!ok) return false;
  p.x = x;
  p.T = int(T), p.b = int(b), p.r = int(r), p.n = int(n), p.P = int(P);
  p.rb_per_tile = int(b / 64);
  p.halves = int(b / kRHalf);
  p.units = (long long)Q * p.rb_per_tile * p.halves;
  cudaError_t e = cudaFuncSetAttribute(blr_recon_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRSmem));
  if (e == cudaSuccess) {
    const int64_t grid = std::min<int64_t>(ctx->sm_count, p.units);
    e = launch_pdl(blr_recon_kernel, dim3(unsigned(grid)), dim3(kRThreads), kRSmem, s, p);
  }
  if (e != cudaSuccess) {
    *st = cuda_fail(ctx, e, "blr_recon_kernel launch");
    return true;
  }
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  *st = LRB_OK;
  return true;
}

}  // namespace lrb
