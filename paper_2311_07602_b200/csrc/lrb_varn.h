// lrb_varn.h — the single-launch variable-size pointer-array kernel
// (lrb_varn.cu): problem descriptor and launch entry shared with the planner.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lrb {

struct ItemDesc;  // lrb_gemm.cuh

constexpr int kVarnMB = 128;    // rows of C per tile (4 warps x 32)
constexpr int kVarnNB = 64;     // max columns of C per tile
constexpr int kVarnKB = 32;     // k chunk per ring slot
constexpr int kVarnStages = 2;  // ring depth (two CTAs per SM)
// Columns past the last full fragment default to one zero-padded fragment:
// the scalar-chain form measured slower at every threshold on cfg4 (rem <= 1:
// 8.49 ms, rem <= 7: 9.10 ms vs 8.29 ms padded; tools/probe_varn.py), so it
// stays an opt-in (LRB_VARN_REM_MAX)
constexpr int kVarnRemMax = 0;

// TMA box width (columns) of an op(B) = N operand for an item with n
// columns: the tile's columns rounded up to the DMMA fragment width
__host__ __device__ __forceinline__ int varn_box_cols(int n) {
  const int c = n < kVarnNB ? n : kVarnNB;
  return (c + 7) / 8 * 8;
}

struct VarnProblem {
  const ItemDesc* items;
  const uint64_t* tiles;       // (item << 32) | (ti << 16) | tj, in claim order
  const CUtensorMap* maps;     // 2 per item (A, B), 3-D with z extent 1
  int64_t num_tiles;
  unsigned long long* next;    // [0] ticket counter, [1] finished CTAs (self-resetting)
};

// a_t / b_t: op flags of the column-major view; flags bit 0: beta = 1
cudaError_t launch_varn(int a_t, int b_t, const VarnProblem& p, int flags, int device,
                        int sm_count, cudaStream_t stream, int64_t* grid);

}  // namespace lrb
