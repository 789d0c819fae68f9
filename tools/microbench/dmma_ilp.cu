// DMMA (m8n8k4 .f64) throughput vs warps per SM sub-partition and independent
// accumulators per warp: can ONE warp per sub-partition keep the FP64 tensor
// pipe busy (ping-pong epilogue overlap)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_ilp dmma_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIters = 2048;
template <int NACC>
__global__ void dmma_ilp(double* out, double x) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = x + threadIdx.x, b = x - threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}
template <int NACC>
void run(int sms, double* out, int warps_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int threads = warps_per_sm * 32;
  dmma_ilp<NACC><<<sms, threads>>>(out, 0.5);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) dmma_ilp<NACC><<<sms, threads>>>(out, 0.5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 5.0 * sms * threads / 32 * double(NACC) * kIters * 512.0;
  std::printf("{\"probe\": \"dmma_ilp\", \"warps_per_smsp\": %d, \"acc_per_warp\": %d, \"tflops\": %.2f}\n",
              warps_per_sm / 4, NACC, flops / (ms * 1e-3) / 1e12);
}
int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  for (int w : {4, 8}) {
    run<8>(p.multiProcessorCount, out, w);
    run<16>(p.multiProcessorCount, out, w);
    run<32>(p.multiProcessorCount, out, w);
  }
  return 0;
}
