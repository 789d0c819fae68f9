// lrb_panel.h — host entry of the row-panel kernel (lrb_panel.cu) for
// short-k strided products (op(A) = N in the column-major view, 1 <= k <= 32).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "lrb_gemm.cuh"

namespace lrb {

constexpr int kPanelRows = 256;   // C rows per unit (two 128-row half panels)
constexpr int kPanelCols = 32;    // C columns per streamed chunk
constexpr int kPanelKMax = 32;    // longest inner dimension the kernel holds
constexpr int kPanelStages = 8;   // V chunk ring depth

size_t panel_smem_bytes();
int panel_threads();
// prob: the operand maps encoded with boxes (128 + 4) x 32 (A) and
// (32 + 4) x 32 (B); num_tiles = units = ceil(m / 256) * batch.
cudaError_t launch_panel(int b_t, const StridedProblem& prob, int flags, int device,
                         int sm_count, cudaStream_t stream, int64_t* grid);

}  // namespace lrb
