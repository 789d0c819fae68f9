// write_pat.cu — which store patterns / cache policies approach cudaMemset's
// write rate on B200 (write_bw.cu: memset 7.4 TB/s, every st.global / TMA
// store form 6.1-6.4 TB/s). One JSON line per variant over an 8 GiB buffer.
//
//   stg32            grid-stride st.global.v4.f64 (the write_bw baseline)
//   stg32_blocked    each CTA owns one contiguous slice of the buffer
//   stg32_chunk{K}   CTAs take contiguous K-KiB chunks round-robin
//   stg32_ef / _el / _nalloc   the baseline with an L2 cache-hint policy
//                    (evict_first / evict_last / evict_unchanged)
//   stg32_wt         st.global.wt
//   bulk_ef          cp.async.bulk shared -> global, 16 KB, evict_first hint
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_pat write_pat.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

enum Pol { NONE = 0, EF = 1, EL = 2, NALLOC = 3, WT = 4, CS = 5 };

template <int POL>
__device__ __forceinline__ void store32(double* p, uint64_t pol) {
  if (POL == NONE)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(0.0), "d"(1.0), "d"(2.0),
                 "d"(3.0)
                 : "memory");
  else if (POL == WT)
    asm volatile("st.global.wt.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(0.0), "d"(1.0),
                 "d"(2.0), "d"(3.0)
                 : "memory");
  else if (POL == CS)
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(0.0), "d"(1.0),
                 "d"(2.0), "d"(3.0)
                 : "memory");
  else
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(0.0),
                 "d"(1.0), "d"(2.0), "d"(3.0), "l"(pol)
                 : "memory");
}

template <int POL>
__device__ __forceinline__ uint64_t make_policy() {
  uint64_t pol = 0;
  if (POL == EF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (POL == EL) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (POL == NALLOC)
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// chunk4 = contiguous run, in 32-byte units, a CTA writes before moving on by
// gridDim.x runs (chunk4 == blockDim.x: the plain grid-stride loop)
template <int POL>
__global__ void stg_kernel(double* __restrict__ out, size_t n4, size_t chunk4) {
  const uint64_t pol = make_policy<POL>();
  const size_t chunks = n4 / chunk4;
  for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    double* base = out + 4 * c * chunk4;
    for (size_t i = threadIdx.x; i < chunk4; i += blockDim.x) store32<POL>(base + 4 * i, pol);
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int POL>
__global__ void bulk_kernel(double* __restrict__ out, size_t chunks) {
  extern __shared__ __align__(128) unsigned char smem[];
  for (int i = threadIdx.x; i < 16384 / 8; i += blockDim.x)
    reinterpret_cast<double*>(smem)[i] = double(i);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t pol = make_policy<POL>();
  for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    if (POL == NONE)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(
                       reinterpret_cast<char*>(out) + c * 16384),
                   "r"(su32(smem))
                   : "memory");
    else
      asm volatile(
          "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], 16384, %2;" ::"l"(
              reinterpret_cast<char*>(out) + c * 16384),
          "r"(su32(smem)), "l"(pol)
          : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
static double best_ms(F launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  launch();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < 5; ++i) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  return best;
}

static void line(const char* mode, double bytes, double ms, const char* extra = "") {
  std::printf("{\"mode\": \"%s\", \"gib\": %.2f, \"ms\": %.4f, \"gbs\": %.1f%s}\n", mode,
              bytes / double(1ull << 30), ms, bytes / ms / 1e6, extra);
  std::fflush(stdout);
}

int main() {
  const size_t bytes = size_t(8) << 30;
  double* buf = nullptr;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t n4 = bytes / 32;
  line("memset", double(bytes), best_ms([&] { CK(cudaMemsetAsync(buf, 0, bytes)); }));
  for (int per : {2, 4}) {
    char ex[96];
    const int grid = sms * per;
    std::snprintf(ex, sizeof ex, ", \"ctas_per_sm\": %d", per);
    line("stg32", double(bytes), best_ms([&] { stg_kernel<NONE><<<grid, 256>>>(buf, n4, 256); }),
         ex);
    // one contiguous slice per CTA (the tail past grid * slice is not written: < 0.01 %)
    line("stg32_blocked", double(bytes),
         best_ms([&] { stg_kernel<NONE><<<grid, 256>>>(buf, n4, n4 / grid); }), ex);
    for (int kib : {64, 256, 1024, 4096}) {
      char m[32];
      std::snprintf(m, sizeof m, "stg32_chunk%d", kib);
      line(m, double(bytes),
           best_ms([&] { stg_kernel<NONE><<<grid, 256>>>(buf, n4, size_t(kib) * 32); }), ex);
    }
    line("stg32_ef", double(bytes), best_ms([&] { stg_kernel<EF><<<grid, 256>>>(buf, n4, 256); }),
         ex);
    line("stg32_el", double(bytes), best_ms([&] { stg_kernel<EL><<<grid, 256>>>(buf, n4, 256); }),
         ex);
    line("stg32_eu", double(bytes),
         best_ms([&] { stg_kernel<NALLOC><<<grid, 256>>>(buf, n4, 256); }), ex);
    line("stg32_wt", double(bytes), best_ms([&] { stg_kernel<WT><<<grid, 256>>>(buf, n4, 256); }),
         ex);
    line("stg32_cs", double(bytes), best_ms([&] { stg_kernel<CS><<<grid, 256>>>(buf, n4, 256); }),
         ex);
    line("stg32_ef_chunk1024", double(bytes),
         best_ms([&] { stg_kernel<EF><<<grid, 256>>>(buf, n4, 1024 * 32); }), ex);
  }
  CK(cudaFuncSetAttribute(bulk_kernel<NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  CK(cudaFuncSetAttribute(bulk_kernel<EF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  CK(cudaFuncSetAttribute(bulk_kernel<NALLOC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          16384));
  for (int per : {2, 4}) {
    char ex[64];
    std::snprintf(ex, sizeof ex, ", \"ctas_per_sm\": %d", per);
    line("bulk", double(bytes),
         best_ms([&] { bulk_kernel<NONE><<<sms * per, 32, 16384>>>(buf, bytes / 16384); }), ex);
    line("bulk_ef", double(bytes),
         best_ms([&] { bulk_kernel<EF><<<sms * per, 32, 16384>>>(buf, bytes / 16384); }), ex);
    line("bulk_eu", double(bytes),
         best_ms([&] { bulk_kernel<NALLOC><<<sms * per, 32, 16384>>>(buf, bytes / 16384); }), ex);
  }
  return 0;
}
