// FP64 pipe probes for B200 (sm_100a), second round:
//  (1) do DMMA (mma.sync .f64, tensor pipe) and DFMA (fp64 pipe) add up when one
//      warp interleaves them? (decides whether scalar DFMA chains can take the
//      padded remainder columns of a variable-rank batch for free)
//  (2) the sustained FP64 DMMA rate: back-to-back launches for several seconds,
//      the figure a kernel timed inside a long step sees (power-capped clocks).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
// prints one JSON line per probe
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

constexpr int kIters = 2048;

__device__ __forceinline__ void mma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// per iteration: 8 DMMA (8 x 256 FMA per warp) and NF DFMA per thread (NF x 32 per warp)
template <int NF, bool DMMA>
__global__ void mix(double* out, double x) {
  double acc[8][2];
  double f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = threadIdx.x * 1e-9 + i;
  const double a = x + threadIdx.x, b = x - 1.0;
  for (int it = 0; it < kIters; ++it) {
    if (DMMA) {
#pragma unroll
      for (int i = 0; i < 8; ++i) mma_m8n8k4(acc[i][0], acc[i][1], a + i, b);
    }
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i & 15] = fma(f[i & 15], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NF, bool DMMA>
void run(const char* name, int blocks_per_sm, int threads, int sms, double* out) {
  auto k = mix<NF, DMMA>;
  const int grid = sms * blocks_per_sm;
  k<<<grid, threads>>>(out, 1.0);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 20;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) k<<<grid, threads>>>(out, 1.0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double warps = double(grid) * threads / 32;
  const double fma_dmma = DMMA ? warps * kIters * 8 * 256.0 : 0.0;
  const double fma_dfma = warps * kIters * NF * 32.0;
  const double s = ms * 1e-3 / reps;
  std::printf("{\"probe\": \"%s\", \"dfma_per_8dmma\": %d, \"warps_per_sm\": %d, \"dmma_tflops\": %.2f, "
              "\"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
              name, NF, blocks_per_sm * threads / 32, 2 * fma_dmma / s / 1e12,
              2 * fma_dfma / s / 1e12, 2 * (fma_dmma + fma_dfma) / s / 1e12);
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int sms = p.multiProcessorCount;
  run<0, true>("dmma_only", 2, 128, sms, out);
  run<16, false>("dfma_only", 2, 512, sms, out);
  run<8, true>("mix", 2, 128, sms, out);
  run<16, true>("mix", 2, 128, sms, out);
  run<32, true>("mix", 2, 128, sms, out);
  run<64, true>("mix", 2, 128, sms, out);
  // sustained DMMA: back-to-back launches for ~6 s, rate over the last 3 s
  {
    auto k = mix<0, true>;
    const int grid = sms * 2, threads = 128;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const auto t0 = std::chrono::steady_clock::now();
    double best_sustained = 0;
    int windows = 0;
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 6.0) {
      const int reps = 200;
      CK(cudaEventRecord(e0));
      for (int r = 0; r < reps; ++r) k<<<grid, threads>>>(out, 1.0);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double tf = 2.0 * grid * threads / 32 * kIters * 8 * 256.0 * reps / (ms * 1e-3) / 1e12;
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > 3.0) {
        best_sustained += tf;
        ++windows;
      }
    }
    std::printf("{\"probe\": \"dmma_sustained\", \"seconds\": 6, \"tflops\": %.2f, \"windows\": %d}\n",
                windows ? best_sustained / windows : 0.0, windows);
  }
  return 0;
}
