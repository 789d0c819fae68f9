// Streaming-read bandwidth of a TMA bulk-copy (cp.async.bulk) smem ring vs
// copy size, stage size, ring depth and CTAs/SM — the feed of the skinny
// (HBM-bound) GEMM variants. Consumers only wait + release: no math.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw bulk_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" :: "r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(dst)), "l"(src), "r"(n), "r"(su32(bar)) : "memory"); }

// producer warp (last) + CONS consumer warps. Each CTA streams `chunks` chunks
// of `stage_bytes` made of copies of `copy_bytes` from a grid-strided range.
__global__ void stream_kernel(const char* __restrict__ src, size_t total_bytes, int stage_bytes,
                              int copy_bytes, int stages, int cons, double* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(stages) * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cons); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t nchunks = total_bytes / stage_bytes;
  if (warp == cons) {
    int st = 0; uint32_t ph = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mbar_wait(&empty[st], ph ^ 1);
      const char* base = src + c * size_t(stage_bytes);
      unsigned char* dst = smem + size_t(st) * stage_bytes;
      const int ncopies = stage_bytes / copy_bytes;
      if (lane == 0) mbar_expect(&full[st], stage_bytes);
      __syncwarp();
      for (int i = lane; i < ncopies; i += 32) bulk(dst + i * copy_bytes, base + size_t(i) * copy_bytes, copy_bytes, &full[st]);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  double acc = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mbar_wait(&full[st], ph);
    acc += reinterpret_cast<const double*>(smem + size_t(st) * stage_bytes)[lane + 32 * warp];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (++st == stages) { st = 0; ph ^= 1; }
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const size_t bytes = size_t(8) << 30;
  char* src; CK(cudaMalloc(&src, bytes)); CK(cudaMemset(src, 1, bytes));
  double* sink; CK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  struct P { int stage, copy, stages, ctas, cons; };
  std::vector<P> ps;
  for (int copy : {128, 256, 512, 1024, 2048, 4096, 16384})
    for (int stage : {8192, 16384, 32768})
      for (int stages : {2, 4, 6})
        for (int ctas : {1, 2, 4}) {
          if (copy > stage) continue;
          size_t smem = size_t(stage) * stages + 16 * stages + 256;
          if (smem * ctas > 220 * 1024) continue;
          ps.push_back({stage, copy, stages, ctas, 4});
        }
  for (const P& p : ps) {
    size_t smem = size_t(p.stage) * p.stages + 16 * p.stages + 256;
    int grid = prop.multiProcessorCount * p.ctas;
    int threads = (p.cons + 1) * 32;
    stream_kernel<<<grid, threads, smem>>>(src, bytes, p.stage, p.copy, p.stages, p.cons, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) stream_kernel<<<grid, threads, smem>>>(src, bytes, p.stage, p.copy, p.stages, p.cons, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double gbs = 3.0 * bytes / (ms * 1e-3) / 1e9;
    std::printf("{\"copy\": %d, \"stage\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"inflight_kb_per_sm\": %d, \"gbs\": %.1f}\n",
                p.copy, p.stage, p.stages, p.ctas, p.stage * p.stages * p.ctas / 1024, gbs);
  }
  return 0;
}
