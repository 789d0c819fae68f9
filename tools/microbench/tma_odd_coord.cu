// tma_odd_coord.cu — does a tiled TMA load of FP64 accept an ODD inner
// coordinate (a box whose first element is only 8-byte aligned)? The pair
// view proposed for odd leading dimensions (item 0)
// needs it: columns kk and kk + 1 of a column-major operand with odd ld form
// one row of 2 ld doubles, and the odd column's box starts at inner ld + i0.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_odd_coord tma_odd_coord.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, int x, int y, double* out) {
  __shared__ __align__(128) double box[16 * 4];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar)),
                 "r"(16 * 4 * 8)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"((uint32_t)__cvta_generic_to_shared(box)),
        "l"(&map), "r"(x), "r"(y), "r"((uint32_t)__cvta_generic_to_shared(&bar))
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"((uint32_t)__cvta_generic_to_shared(&bar))
          : "memory");
    for (int i = 0; i < 64; ++i) out[i] = box[i];
  }
}

int main() {
  const int ld = 33, pairs = 8;  // 16 columns of an odd-ld column-major operand as 8 rows of 2 ld
  std::vector<double> h(size_t(2) * ld * pairs);
  for (size_t i = 0; i < h.size(); ++i) h[i] = double(i);
  double *d = nullptr, *o = nullptr;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 64 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap map;
  cuuint64_t dims[2] = {cuuint64_t(2 * ld), cuuint64_t(pairs)};
  cuuint64_t strides[1] = {cuuint64_t(2 * ld) * 8};  // 528 bytes: a 16-byte multiple
  cuuint32_t box[2] = {16, 4}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("{\"encode\": %d", int(r));
  if (r != CUDA_SUCCESS) {
    std::printf("}\n");
    return 0;
  }
  for (int x : {0, 1, ld, ld + 5}) {  // even, odd, the odd column's start, odd column + odd offset
    cudaMemset(o, 0, 64 * 8);
    probe<<<1, 32>>>(map, x, 2, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> g(64);
    cudaMemcpy(g.data(), o, 64 * 8, cudaMemcpyDeviceToHost);
    bool ok = e == cudaSuccess;
    for (int row = 0; row < 4 && ok; ++row)
      for (int c = 0; c < 16; ++c) ok = ok && g[row * 16 + c] == double((2 + row) * 2 * ld + x + c);
    std::printf(", \"x%d\": \"%s\"", x, e != cudaSuccess ? cudaGetErrorString(e) : ok ? "exact" : "wrong data");
    if (e != cudaSuccess) break;
  }
  std::printf("}\n");
  return 0;
}
