// FP64 peak probes for B200 (sm_100a): DFMA vs DMMA (mma.sync .f64) throughput,
// DMMA rounding behaviour vs a sequential FMA chain, and HBM stream bandwidth.
// Used once to pick the FP64 roofline denominator and the kernel family; results
// are committed under profiles/.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

constexpr int kIters = 4096;

__global__ void dfma_peak(double* out, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void mma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k4(double (&d)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma_m16n8k16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int KIND>
__global__ void dmma_peak(double* out, double x) {
  // 8 independent accumulator tiles per warp
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = x + threadIdx.x + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = x - i;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) { double d2[2] = {acc[i][0], acc[i][1]}; mma_m8n8k4(d2, a[i], b[0]); acc[i][0] = d2[0]; acc[i][1] = d2[1]; }
      if (KIND == 1) { mma_m16n8k4(acc[i], a[i], a[(i + 1) & 7], b[0]); }
      if (KIND == 2) { double aa[4] = {a[0], a[1], a[2], a[3]}; double bb[2] = {b[0], b[1]}; mma_m16n8k8(acc[i], aa, bb); }
      if (KIND == 3) { mma_m16n8k16(acc[i], a, b); }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// rounding probe: one m8n8k4 with given A (8x4 row), B (4x8 col), C (8x8)
__global__ void dmma_probe(const double* A, const double* B, const double* C, double* D) {
  int l = threadIdx.x, g = l >> 2, t = l & 3;
  double a = A[g * 4 + t];
  double b = B[t * 8 + g];  // B stored row-major 4x8: B[k][n]
  double d[2] = {C[g * 8 + 2 * t], C[g * 8 + 2 * t + 1]};
  mma_m8n8k4(d, a, b);
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
}
// m16n8k16 probe: A 16x16 row-major, B 16x8 row-major (B[k][n]), C/D 16x8 row-major
__global__ void dmma16_probe(const double* A, const double* B, const double* C, double* D) {
  int l = threadIdx.x, g = l >> 2, t = l & 3;
  double a[8], b[4], d[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) { int r = g + 8 * (i & 1); int c = t + 4 * (i >> 1); a[i] = A[r * 16 + c]; }
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  d[0] = C[g * 8 + 2 * t]; d[1] = C[g * 8 + 2 * t + 1];
  d[2] = C[(g + 8) * 8 + 2 * t]; d[3] = C[(g + 8) * 8 + 2 * t + 1];
  mma_m16n8k16(d, a, b);
  D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2]; D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

__global__ void read_bw(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}
__global__ void write_bw(double2* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_double2(1.0, 2.0));
}
__global__ void copy_bw(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

static uint64_t rng_state = 88172645463325252ull;
static double urand() {
  rng_state ^= rng_state << 13; rng_state ^= rng_state >> 7; rng_state ^= rng_state << 17;
  return (double)(rng_state >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  std::printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d}\n", prop.name,
              prop.multiProcessorCount, clk, prop.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = prop.multiProcessorCount;

  // DFMA
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    dfma_peak<<<blocks, threads>>>(out, 1.0000001, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dfma_peak<<<blocks, threads>>>(out, 1.0000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * threads * 16.0 * kIters * 2.0;
    std::printf("{\"probe\": \"dfma\", \"threads\": %d, \"tflops\": %.2f}\n", threads, flops / (ms * 1e-3) / 1e12);
  }
  // DMMA
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double fl[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int kind = 0; kind < 4; ++kind) {
    for (int warps : {4, 8, 16}) {
      int threads = warps * 32, blocks = sms * 2;
      auto launch = [&]() {
        if (kind == 0) dmma_peak<0><<<blocks, threads>>>(out, 0.5);
        if (kind == 1) dmma_peak<1><<<blocks, threads>>>(out, 0.5);
        if (kind == 2) dmma_peak<2><<<blocks, threads>>>(out, 0.5);
        if (kind == 3) dmma_peak<3><<<blocks, threads>>>(out, 0.5);
      };
      launch(); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 5.0 * blocks * warps * 8.0 * (kIters / 4) * fl[kind] * 2.0;
      std::printf("{\"probe\": \"dmma_%s\", \"warps_per_cta\": %d, \"tflops\": %.2f}\n", names[kind], warps,
                  flops / (ms * 1e-3) / 1e12);
    }
  }
  // DMMA throughput vs warps per SM sub-partition (one CTA per SM)
  for (int warps : {4, 8, 12, 16}) {
    int threads = warps * 32, blocks = sms;
    dmma_peak<0><<<blocks, threads>>>(out, 0.5);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dmma_peak<0><<<blocks, threads>>>(out, 0.5);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * warps * 8.0 * (kIters / 4) * fl[0] * 2.0;
    std::printf("{\"probe\": \"dmma_m8n8k4_per_smsp\", \"warps_per_smsp\": %d, \"tflops\": %.2f}\n",
                warps / 4, flops / (ms * 1e-3) / 1e12);
  }
  // DMMA rounding probe (m8n8k4 and m16n8k16) vs sequential FMA chain
  {
    const int trials = 2000;
    std::vector<double> A(16 * 16), B(16 * 8), C(16 * 8), D(16 * 8);
    double *dA, *dB, *dC, *dD;
    CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8));
    CK(cudaMalloc(&dC, C.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
    long seq_mismatch4 = 0, seq_mismatch16 = 0, total4 = 0, total16 = 0;
    for (int tr = 0; tr < trials; ++tr) {
      // scale by random exponents to expose rounding differences
      for (auto& v : A) v = urand() * std::ldexp(1.0, (int)(urand() * 20));
      for (auto& v : B) v = urand() * std::ldexp(1.0, (int)(urand() * 20));
      for (auto& v : C) v = urand() * std::ldexp(1.0, (int)(urand() * 20));
      // m8n8k4: A 8x4 row-major, B 4x8 row-major, C 8x8
      CK(cudaMemcpy(dA, A.data(), 32 * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dB, B.data(), 32 * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dC, C.data(), 64 * 8, cudaMemcpyHostToDevice));
      dmma_probe<<<1, 32>>>(dA, dB, dC, dD);
      CK(cudaMemcpy(D.data(), dD, 64 * 8, cudaMemcpyDeviceToHost));
      for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) {
        double s = C[i * 8 + j];
        for (int p = 0; p < 4; ++p) s = std::fma(A[i * 4 + p], B[p * 8 + j], s);
        seq_mismatch4 += (s != D[i * 8 + j]); ++total4;
      }
      CK(cudaMemcpy(dA, A.data(), 256 * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dB, B.data(), 128 * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dC, C.data(), 128 * 8, cudaMemcpyHostToDevice));
      dmma16_probe<<<1, 32>>>(dA, dB, dC, dD);
      CK(cudaMemcpy(D.data(), dD, 128 * 8, cudaMemcpyDeviceToHost));
      for (int i = 0; i < 16; ++i) for (int j = 0; j < 8; ++j) {
        double s = C[i * 8 + j];
        for (int p = 0; p < 16; ++p) s = std::fma(A[i * 16 + p], B[p * 8 + j], s);
        seq_mismatch16 += (s != D[i * 8 + j]); ++total16;
      }
    }
    std::printf("{\"probe\": \"dmma_rounding\", \"m8n8k4_mismatch_vs_fma_chain\": %ld, \"of\": %ld, "
                "\"m16n8k16_mismatch_vs_fma_chain\": %ld, \"of16\": %ld}\n",
                seq_mismatch4, total4, seq_mismatch16, total16);
  }
  // HBM
  {
    size_t bytes = size_t(4) << 30;  // 4 GiB
    double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
    size_t n = bytes / 16;
    for (int mult : {4, 8, 16}) {
      int blocks = sms * mult, threads = 256;
      float ms;
      read_bw<<<blocks, threads>>>(a, n, out); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); for (int r = 0; r < 5; ++r) read_bw<<<blocks, threads>>>(a, n, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double rd = 5.0 * bytes / (ms * 1e-3) / 1e9;
      write_bw<<<blocks, threads>>>(b, n); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); for (int r = 0; r < 5; ++r) write_bw<<<blocks, threads>>>(b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double wr = 5.0 * bytes / (ms * 1e-3) / 1e9;
      copy_bw<<<blocks, threads>>>(a, b, n); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copy_bw<<<blocks, threads>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double cp = 5.0 * 2.0 * bytes / (ms * 1e-3) / 1e9;
      std::printf("{\"probe\": \"hbm\", \"blocks_per_sm\": %d, \"read_gbs\": %.1f, \"write_gbs\": %.1f, \"copy_gbs\": %.1f}\n",
                  mult * threads / 256, rd, wr, cp);
    }
  }
  return 0;
}
