// Write-stream bandwidth of B200 HBM3e: what a kernel whose bytes are almost
// all output (the expansions, the dense reconstruction, cfg2's C) can reach.
// One JSON line per mode, best of 5 launches timed with CUDA events over an
// 8 GiB buffer (64x L2):
//   memset       cudaMemsetAsync
//   stg16 / stg32  grid-stride st.global.v2.f64 / st.global.v4.f64 (16 / 32 B per lane)
//   stg32_cs     the same with the streaming (.cs) hint
//   tma_bulk     cp.async.bulk.global.shared::cta of 16 KB smem chunks, one
//                elected lane per CTA, 4 bulk groups in flight
//   tma_box16    cp.async.bulk.tensor.2d of 16 x 16 FP64 boxes (2 KB, 128-byte
//                swizzle) from per-warp staging, the expansion kernel's store
//                pattern: each warp writes a 16-row x 32-column piece of
//                64 x 256 units, rows of `row_doubles`
//   read         grid-stride ld.global.v4.f64 (sum into a sink), for scale
//   copy         read + write of 4 GiB each (bytes counted both ways, like
//                MEASURED_PEAKS.json's copy figure)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_bw write_bw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void stg16_kernel(double* __restrict__ out, size_t n2) {
  const double2 z = make_double2(0.0, 1.0);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2;
       i += size_t(gridDim.x) * blockDim.x)
    reinterpret_cast<double2*>(out)[i] = z;
}

template <bool CS>
__global__ void stg32_kernel(double* __restrict__ out, size_t n4) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
       i += size_t(gridDim.x) * blockDim.x) {
    double* p = out + 4 * i;
    if (CS)
      asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(0.0), "d"(1.0),
                   "d"(2.0), "d"(3.0)
                   : "memory");
    else
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(0.0), "d"(1.0),
                   "d"(2.0), "d"(3.0)
                   : "memory");
  }
}

__global__ void read_kernel(const double* __restrict__ in, size_t n4, double* sink) {
  double s = 0.0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
       i += size_t(gridDim.x) * blockDim.x) {
    double a, b, c, d;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(in + 4 * i));
    s += a + b + c + d;
  }
  if (s == 12345.678) *sink = s;
}

__global__ void copy_kernel(const double* __restrict__ in, double* __restrict__ out, size_t n4) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
       i += size_t(gridDim.x) * blockDim.x) {
    double a, b, c, d;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(in + 4 * i));
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(out + 4 * i), "d"(a), "d"(b),
                 "d"(c), "d"(d)
                 : "memory");
  }
}

// one elected lane per CTA issues 16 KB bulk stores from a zeroed smem slab
__global__ void tma_bulk_kernel(double* __restrict__ out, size_t chunks) {
  extern __shared__ __align__(1024) unsigned char smem[];
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(
                     reinterpret_cast<char*>(out) + c * 16384),
                 "r"(su32(smem))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the expansion kernel's store pattern: 8 warps, each stages a 16 x 32 piece
// (two 16 x 16 boxes) per 64 x 64 block of a 64-row x 256-column unit
struct BoxArgs {
  CUtensorMap map;
  int units, unit_cols, rows;  // units over a (rows x row_doubles) matrix
};
__global__ void __launch_bounds__(256, 1) tma_box_kernel(const __grid_constant__ BoxArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* st = reinterpret_cast<double*>(smem) + warp * 4 * 512;  // 4 sub-blocks of 16 x 32
  for (int i = lane; i < 4 * 512; i += 32) st[i] = double(i);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int row0 = (warp & 3) * 16, colw = (warp >> 2) * 32;
  const int per_row = a.unit_cols / 256;
  int buf = 0;
  for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
    const int ub = u / per_row, uh = u - ub * per_row;
    for (int cb = 0; cb < 4; ++cb) {
      if (lane == 0) {
        const double* src = st + buf * 512;
        const int x0 = uh * 256 + cb * 64 + colw, y0 = ub * 64 + row0;
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::
                "l"(&a.map),
            "r"(su32(src)), "r"(x0), "r"(y0)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::
                "l"(&a.map),
            "r"(su32(src + 256)), "r"(x0 + 16), "r"(y0)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
      }
      __syncwarp();
      buf = (buf + 1) & 3;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int sm_count() {
  int d = 0, n = 0;
  CK(cudaGetDevice(&d));
  CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d));
  return n;
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
  double* sink = nullptr;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 0, bytes));
  const int sms = sm_count();
  const size_t n = bytes / 8;

  line("memset", double(bytes), best_ms([&] { CK(cudaMemsetAsync(buf, 0, bytes)); }));
  for (int per : {2, 4, 8}) {
    char ex[64];
    std::snprintf(ex, sizeof ex, ", \"ctas_per_sm\": %d", per);
    line("stg16", double(bytes),
         best_ms([&] { stg16_kernel<<<sms * per, 256>>>(buf, n / 2); }), ex);
    line("stg32", double(bytes),
         best_ms([&] { stg32_kernel<false><<<sms * per, 256>>>(buf, n / 4); }), ex);
    line("stg32_cs", double(bytes),
         best_ms([&] { stg32_kernel<true><<<sms * per, 256>>>(buf, n / 4); }), ex);
    line("read", double(bytes),
         best_ms([&] { read_kernel<<<sms * per, 256>>>(buf, n / 4, sink); }), ex);
    line("copy", double(bytes),
         best_ms([&] { copy_kernel<<<sms * per, 256>>>(buf, buf + n / 2, n / 8); }), ex);
  }
  CK(cudaFuncSetAttribute(tma_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  for (int per : {1, 2, 4, 8}) {
    char ex[64];
    std::snprintf(ex, sizeof ex, ", \"ctas_per_sm\": %d", per);
    line("tma_bulk", double(bytes),
         best_ms([&] { tma_bulk_kernel<<<sms * per, 32, 16384>>>(buf, bytes / 16384); }), ex);
  }
  // the expansion store pattern over an (rows x row_doubles) row-major matrix
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr));
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  }
  CK(cudaFuncSetAttribute(tma_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          8 * 4 * 512 * 8));
  for (int row_doubles : {512, 4096, 16384}) {
    const int rows = int(n / row_doubles);
    BoxArgs a;
    cuuint64_t dims[2] = {cuuint64_t(row_doubles), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(row_doubles) * 8};
    cuuint32_t box[2] = {16, 16};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      std::fprintf(stderr, "encode failed\n");
      return 1;
    }
    a.rows = rows;
    a.unit_cols = row_doubles;
    a.units = (rows / 64) * (row_doubles / 256);
    char ex[96];
    std::snprintf(ex, sizeof ex, ", \"row_doubles\": %d, \"ctas_per_sm\": 1", row_doubles);
    line("tma_box16", double(size_t(a.units) * 64 * 256 * 8),
         best_ms([&] { tma_box_kernel<<<sms, 256, 8 * 4 * 512 * 8>>>(a); }), ex);
  }
  return 0;
}
