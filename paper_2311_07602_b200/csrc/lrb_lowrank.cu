// lrb_lowrank.cu — the paper's batched low-rank product on B200.
//
//   G_i = A_X_i (A_Vt_i B_U_i) B_X_i        (arXiv 2311.07602, Algorithm 1)
//
// over a LowRankBatch: every matrix row-major, each role packed
// contiguously (item i at base + i*rows*cols), rank_a == rank_b == r
// (reference low_rank.hpp:109-176; drivers fused_multiply / packed_multiply,
// kernels.hpp:131-349; oracle low_rank_multiply_reference_raw,
// low_rank.hpp:73-87). Each of the three products is an in-order FMA chain
// over its inner index, so G is bitwise the reference oracle's three naive
// products computed with fused multiply-adds.
//
// Fast path (r <= 32, even block, 16-B aligned roles): one warp per item,
// four items per CTA, persistent CTAs. Odd ranks included: B_U's rows are
// then r doubles, not a 16-byte multiple, and the tensor map views each item
// as b/2 rows of 2r instead (LrCfg::P2; the columns past r are masked).
//   * C^T = B_U^T A_Vt^T on FP64 DMMA with k ascending; the A_Vt and B_U
//     chunks of the CTA's four items arrive with ONE 3-D TMA box each
//     (z = item), padded so fragment loads are bank-conflict free.
//   * E = A_X C and G = E B_X straight from the accumulators: a lane's
//     accumulator pair already shares the column the next product needs as an
//     operand, so four quad-local shuffles per k-block turn accumulators into
//     MMA operands — no shared-memory round trip; G is stored once.
// r > 32: three batched GEMMs (lrb_dgemm_strided_batched's kernels) with the
// intermediates in the context workspace. Other shapes: a plain per-item
// kernel (same FMA chains).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "lrb_dispatch.cuh"
#include "lrb_internal.h"

namespace lrb {

// declared in lrb_api.cu
lrb_status run_strided_rowmajor(lrb_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                                int64_t sA, const double* B, int64_t sB, double* C, int64_t sC,
                                int64_t batch, cudaStream_t stream);
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
// lrb_lowrank_big.cu: ranks 64 / 96 / 128 in one launch, T and E on chip
bool lowrank_big_eligible(int64_t batch, int64_t block, int64_t rank, const void* a_vt,
                          const void* b_u, const void* a_x, const void* b_x);
lrb_status run_lowrank_big(lrb_ctx* ctx, int64_t batch, int64_t block, int64_t rank,
                           const double* a_vt, const double* b_u, const double* a_x,
                           const double* b_x, double* g, cudaStream_t s);

template <int R>
struct LrCfg {
  static constexpr int G = 4;  // items per CTA, one warp each
  // r = 8: a fifth warp issues the refills behind empty barriers (the item
  // warps' 4-stage ring turns over fastest there): 0.95-0.98 -> 1.00-1.02 of
  // HBM. r = 16 measured within +-1% either way, and r = 32 needs 255
  // registers: both keep the last-warp-out refill
  static constexpr bool PROD = R <= 8;
  static constexpr int THREADS = 32 * G + (PROD ? 32 : 0);
  static constexpr int KB = (R >= 32) ? 16 : 32;
  static constexpr int STAGES = (R <= 8) ? 4 : 2;
  static constexpr int F = R / 8;
  static constexpr int PK = KB + 4;  // A_Vt tile [m][kk]
  static constexpr int PR = R + 4;   // B_U tile  [kk][n]
  static constexpr int AV = PK * R;  // per item: box (KB+4, R, G)
  static constexpr int BU = PR * KB; // per item: box (R+4, KB, G)
  // odd ranks (PAIR): B_U's rows are r doubles, not a 16-byte multiple, so
  // the map views each item as b/2 rows of 2r (rows kk, kk+1 side by side):
  // box (2R+4, KB/2, G). Element (kk, n) sits at (kk/2) P2 + (kk%2) r + n;
  // past 2r the box is zero-filled, so n >= r reads zeros on odd kk and the
  // neighbouring row (masked to zero) on even kk. It fits B_U's buffer.
  static constexpr int P2 = 2 * R + 4;
  static constexpr int BUP = P2 * (KB / 2);
  static_assert(BUP <= BU, "the paired box fits the B_U buffer");
  static constexpr int AV_ELEMS = round_up_c(AV * G, 16);
  static constexpr int BU_ELEMS = round_up_c(BU * G, 16);
  static constexpr int STAGE = AV_ELEMS + BU_ELEMS;
  static constexpr size_t SMEM =
      size_t(STAGES) * STAGE * 8 + size_t(STAGES) * 8 + size_t(STAGES) * 4 + 32 +
      (PROD ? size_t(STAGES) * 8 + 8 : 0);
};

struct LrProblem {
  CUtensorMap tmAV;  // (b, r, batch) view of A_Vt
  CUtensorMap tmBU;  // (r, b, batch) view of B_U
  const double* a_vt;
  const double* b_u;
  const double* a_x;
  const double* b_x;
  double* g;
  int64_t batch;
  int block, rank;
  int64_t groups;  // ceil(batch / G)
};

template <class Cf, bool PAIR>
__device__ __forceinline__ void lr_issue(const LrProblem& p, double* smem, uint64_t* full,
                                         IssueState* st, int stage, int lane) {
  long long t_ll = 0;
  int k0 = 0;
  if (lane == 0) {
    t_ll = st->t;
    k0 = st->k0;
  }
  const int64_t t = __shfl_sync(0xffffffffu, t_ll, 0);
  k0 = __shfl_sync(0xffffffffu, k0, 0);
  if (t >= p.groups) return;
  if (lane == 0) {
    double* av = smem + size_t(stage) * Cf::STAGE;
    double* bu = av + Cf::AV_ELEMS;
    fence_proxy_async_smem();
    // A_Vt and B_U are read once, but A_Vt's box is k-contiguous: its pitch
    // pad reads the next chunk's first k-columns, which must stay in L2
    // (measured: r = 16/32 rows +3-6%; r = 8, where the pad is 1/9 of the
    // box and the ring is 4 deep, stays evict-first)
    const uint64_t pol_av = (Cf::F >= 2) ? policy_evict_normal() : policy_evict_first();
    const uint64_t pol_bu = policy_evict_first();
    mbar_arrive_expect_tx(&full[stage], uint32_t(Cf::AV + (PAIR ? Cf::BUP : Cf::BU)) * Cf::G * 8u);
    const int z = static_cast<int>(t * Cf::G);
    tma_load_3d(av, &p.tmAV, k0, 0, z, &full[stage], pol_av);
    tma_load_3d(bu, &p.tmBU, 0, PAIR ? k0 / 2 : k0, z, &full[stage], pol_bu);
    int nk0 = k0 + Cf::KB;
    int64_t nt = t;
    if (nk0 >= p.block) {
      nk0 = 0;
      nt = t + gridDim.x;
    }
    st->t = nt;
    st->k0 = nk0;
  }
  __syncwarp();
}

template <int R, bool PAIR>
__global__ void __launch_bounds__(LrCfg<R>::THREADS, 2)
    lrb_lowrank_kernel(const __grid_constant__ LrProblem p) {
  using Cf = LrCfg<R>;
  constexpr int F = Cf::F, KB = Cf::KB, STAGES = Cf::STAGES;
  pdl_entry();
  extern __shared__ __align__(1024) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * Cf::STAGE);
  IssueState* st = reinterpret_cast<IssueState*>(full + STAGES);
  int* released = reinterpret_cast<int*>(st + 1);
  uint64_t* empty = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(released + STAGES) + 7) & ~uintptr_t(7));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int r = p.rank;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
      if (Cf::PROD) mbar_init(&empty[s], Cf::G);
    }
    st->t = blockIdx.x;
    st->k0 = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (Cf::PROD) {
    if (warp == Cf::G) {
      // producer: every (group, k-chunk) of the CTA in order, each into its
      // slot once the four item warps have released it
      int q = 0;
#pragma unroll 1
      for (;; ++q) {
        const int s = q % STAGES;
        if (q >= STAGES) {
          if (lane == 0) mbar_wait(&empty[s], ((q / STAGES) - 1) & 1);
          __syncwarp();
        }
        long long t_ll = 0;
        if (lane == 0) t_ll = st->t;
        if (__shfl_sync(0xffffffffu, t_ll, 0) >= p.groups) break;
        lr_issue<Cf, PAIR>(p, smem, full, st, s, lane);
      }
      return;
    }
  } else {
    if (warp == 0)
      for (int s = 0; s < STAGES; ++s) lr_issue<Cf, PAIR>(p, smem, full, st, s, lane);
  }

  int stage = 0;
  uint32_t phase = 0;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < p.groups; t += gridDim.x) {
    const int64_t item = t * Cf::G + warp;
    if (item < p.batch) {
      // the epilogue reads this item's A_X and B_X (2 r^2 doubles) with its
      // latency exposed: start them towards L2 while the main loop runs
      const char* pax = reinterpret_cast<const char*>(p.a_x + item * int64_t(r) * r);
      const char* pbx = reinterpret_cast<const char*>(p.b_x + item * int64_t(r) * r);
      const int bytes = r * r * 8;
      for (int off = lane * 128; off < bytes; off += 32 * 128) {
        prefetch_l2(pax + off);
        prefetch_l2(pbx + off);
      }
    }
    // acc[fn][fm][c] = C[m = fm*8 + 2tq + c][n = fn*8 + g]   (D of C^T = B_U^T A_Vt^T)
    double acc[F][F][2];
#pragma unroll
    for (int a = 0; a < F; ++a)
#pragma unroll
      for (int b = 0; b < F; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll 1
    for (int k0 = 0; k0 < p.block; k0 += KB) {
      const int kvalid = min(KB, p.block - k0);
      mbar_wait(&full[stage], phase);
      const double* As = smem + size_t(stage) * Cf::STAGE + warp * Cf::AV;       // [m][kk]
      const double* Bs = smem + size_t(stage) * Cf::STAGE + Cf::AV_ELEMS +
                         warp * (PAIR ? Cf::BUP : Cf::BU);  // [kk][n]
      // B_U[kk][n] (PAIR: the row-pair layout, columns past r masked)
      auto bu_at = [&](int kk, int n) -> double {
        if constexpr (PAIR) {
          const double v = Bs[(kk >> 1) * Cf::P2 + (kk & 1) * r + n];
          return ((kk & 1) || n < r) ? v : 0.0;
        } else {
          return Bs[kk * Cf::PR + n];
        }
      };
      const int nq = kvalid >> 2;
#pragma unroll 4
      for (int kq = 0; kq < nq; ++kq) {
        const int kk = kq * 4 + tq;
        double af[F], bf[F];
#pragma unroll
        for (int fn = 0; fn < F; ++fn) af[fn] = bu_at(kk, fn * 8 + g);  // B_U[kk][n]
#pragma unroll
        for (int fm = 0; fm < F; ++fm) bf[fm] = As[(fm * 8 + g) * Cf::PK + kk];  // A_Vt[m][kk]
#pragma unroll
        for (int fn = 0; fn < F; ++fn)
#pragma unroll
          for (int fm = 0; fm < F; ++fm) dmma_8x8x4(acc[fn][fm][0], acc[fn][fm][1], af[fn], bf[fm]);
      }
#pragma unroll 1
      for (int kk = nq * 4; kk < kvalid; ++kk) {
#pragma unroll
        for (int fn = 0; fn < F; ++fn) {
          const double bv = bu_at(kk, fn * 8 + g);
#pragma unroll
          for (int fm = 0; fm < F; ++fm)
#pragma unroll
            for (int c = 0; c < 2; ++c)
              acc[fn][fm][c] = fma(As[(fm * 8 + 2 * tq + c) * Cf::PK + kk], bv, acc[fn][fm][c]);
        }
      }
      __syncwarp();
      if constexpr (Cf::PROD) {
        if (lane == 0) mbar_arrive(&empty[stage]);
      } else {
        int last = 0;
        if (lane == 0) {
          last = (atom_add_acq_rel_cta(&released[stage], 1) == Cf::G - 1);
          if (last) released[stage] = 0;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) lr_issue<Cf, PAIR>(p, smem, full, st, stage, lane);
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (item >= p.batch) continue;  // warp-uniform

    const double* ax = p.a_x + item * int64_t(r) * r;
    const double* bx = p.b_x + item * int64_t(r) * r;
    // quad-local source lane of k-block half h: C[m0 + tq][.] lives in lane
    // (g, 2h + tq/2), element tq & 1
    // ---- E = A_X C:  e[fx][fn][c] = E[x = fx*8 + g][n = fn*8 + 2tq + c]
    double e[F][F][2];
#pragma unroll
    for (int a = 0; a < F; ++a)
#pragma unroll
      for (int b = 0; b < F; ++b) e[a][b][0] = e[a][b][1] = 0.0;
    // k-blocks (fm, h) ascending outermost: each A_X value is loaded once and
    // every accumulator still receives its DMMAs in ascending m order
#pragma unroll
    for (int fm = 0; fm < F; ++fm)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int src = g * 4 + 2 * h + (tq >> 1);
        const int mcol = fm * 8 + 4 * h + tq;  // m
        double a[F];
#pragma unroll
        for (int fx = 0; fx < F; ++fx) {
          const int x = fx * 8 + g;
          a[fx] = (x < r && mcol < r) ? __ldg(ax + x * r + mcol) : 0.0;  // A_X[x][m]
        }
#pragma unroll
        for (int fn = 0; fn < F; ++fn) {
          const double v0 = __shfl_sync(0xffffffffu, acc[fn][fm][0], src);
          const double v1 = __shfl_sync(0xffffffffu, acc[fn][fm][1], src);
          const double cb = (tq & 1) ? v1 : v0;  // B-operand C[m0 + tq][fn*8 + g]
#pragma unroll
          for (int fx = 0; fx < F; ++fx) dmma_8x8x4(e[fx][fn][0], e[fx][fn][1], a[fx], cb);
        }
      }
    // ---- G = E B_X:  o[fx][fy][c] = G[x = fx*8 + g][y = fy*8 + 2tq + c]
    double o[F][F][2];
#pragma unroll
    for (int a = 0; a < F; ++a)
#pragma unroll
      for (int b = 0; b < F; ++b) o[a][b][0] = o[a][b][1] = 0.0;
    // k-blocks (fn, h) ascending outermost: each B_X value is loaded once
#pragma unroll
    for (int fn = 0; fn < F; ++fn)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int src = g * 4 + 2 * h + (tq >> 1);
        const int nrow = fn * 8 + 4 * h + tq;  // n
        double b[F];
#pragma unroll
        for (int fy = 0; fy < F; ++fy) {
          const int y = fy * 8 + g;
          b[fy] = (nrow < r && y < r) ? __ldg(bx + nrow * r + y) : 0.0;  // B_X[n][y]
        }
#pragma unroll
        for (int fx = 0; fx < F; ++fx) {
          const double v0 = __shfl_sync(0xffffffffu, e[fx][fn][0], src);
          const double v1 = __shfl_sync(0xffffffffu, e[fx][fn][1], src);
          const double ea = (tq & 1) ? v1 : v0;  // A-operand E[fx*8 + g][n0 + tq]
#pragma unroll
          for (int fy = 0; fy < F; ++fy) dmma_8x8x4(o[fx][fy][0], o[fx][fy][1], ea, b[fy]);
        }
      }
    // ---- store G once (row-major r x r)
    double* gp = p.g + item * int64_t(r) * r;
    const bool vec = ((r & 1) == 0) && ((reinterpret_cast<uintptr_t>(gp) & 15) == 0);
#pragma unroll
    for (int fx = 0; fx < F; ++fx) {
      const int x = fx * 8 + g;
      if (x < r) {
#pragma unroll
        for (int fy = 0; fy < F; ++fy) {
          const int y = fy * 8 + 2 * tq;
          if (vec && y + 1 < r) {
            st_global_v2(gp + x * r + y, o[fx][fy][0], o[fx][fy][1]);
          } else {
            if (y < r) st_global_cs(gp + x * r + y, o[fx][fy][0]);
            if (y + 1 < r) st_global_cs(gp + x * r + y + 1, o[fx][fy][1]);
          }
        }
      }
    }
  }
}

// Any shape: one CTA per item, entries spread over threads, the same three
// in-order FMA chains; intermediates in shared memory (2 r^2 doubles).
__global__ void lrb_lowrank_simple_kernel(const double* __restrict__ a_vt,
                                          const double* __restrict__ b_u,
                                          const double* __restrict__ a_x,
                                          const double* __restrict__ b_x, double* __restrict__ g,
                                          int64_t batch, int block, int rank) {
  pdl_entry();
  extern __shared__ double sm[];
  double* cs = sm;
  double* es = sm + size_t(rank) * rank;
  const int rr = rank * rank;
  for (int64_t item = blockIdx.x; item < batch; item += gridDim.x) {
    const double* av = a_vt + item * int64_t(rank) * block;
    const double* bu = b_u + item * int64_t(block) * rank;
    const double* ax = a_x + item * int64_t(rr);
    const double* bx = b_x + item * int64_t(rr);
    for (int e = threadIdx.x; e < rr; e += blockDim.x) {
      const int m = e / rank, n = e - m * rank;
      double s = 0.0;
      for (int k = 0; k < block; ++k) s = fma(av[int64_t(m) * block + k], bu[int64_t(k) * rank + n], s);
      cs[e] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rr; e += blockDim.x) {
      const int x = e / rank, n = e - x * rank;
      double s = 0.0;
      for (int m = 0; m < rank; ++m) s = fma(ax[x * rank + m], cs[m * rank + n], s);
      es[e] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rr; e += blockDim.x) {
      const int x = e / rank, y = e - x * rank;
      double s = 0.0;
      for (int n = 0; n < rank; ++n) s = fma(es[x * rank + n], bx[n * rank + y], s);
      g[item * int64_t(rr) + e] = s;
    }
    __syncthreads();
  }
}

namespace {

bool encode3(CUtensorMap* map, const double* base, int64_t d0, int64_t d1, int64_t d2,
             int64_t s1, int64_t s2, int b0, int b1, int b2) {
  auto fn = encode_fn();
  if (!fn) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (s1 & 1) || (d2 > 1 && (s2 & 1))) return false;
  cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(d2)};
  cuuint64_t strides[2] = {cuuint64_t(s1 * 8), cuuint64_t((d2 > 1 ? s2 : s1 * d1 + (s1 * d1) % 2) * 8)};
  cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(b1), cuuint32_t(b2)};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int R, bool PAIR>
cudaError_t launch_fast(const LrProblem& p, int device, int sm_count, cudaStream_t s,
                        int64_t* grid_out) {
  using Cf = LrCfg<R>;
  auto kern = lrb_lowrank_kernel<R, PAIR>;
  static int occ_cache[64] = {0};
  int occ = (device >= 0 && device < 64) ? occ_cache[device] : 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(Cf::SMEM));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (device >= 0 && device < 64) occ_cache[device] = occ;
  }
  const int64_t grid = std::min<int64_t>(p.groups, int64_t(sm_count) * occ);
  *grid_out = grid;
  if (grid > 0) return launch_pdl(kern, dim3(unsigned(grid)), dim3(Cf::THREADS), Cf::SMEM, s, p);
  return cudaSuccess;
}

}  // namespace

// 0 fast (TMA + DMMA), 1 three GEMMs, 2 simple kernel
int lowrank_path(int64_t block, int64_t rank, const void* a_vt, const void* b_u) {
  if (rank > 32) return 1;
  const bool aligned = ((reinterpret_cast<uintptr_t>(a_vt) | reinterpret_cast<uintptr_t>(b_u)) & 15) == 0;
  // (odd ranks too: B_U is then mapped as row pairs, LrCfg::P2)
  if ((block & 1) == 0 && aligned && encode_fn()) return 0;
  return 2;
}

lrb_status run_lowrank(lrb_ctx* ctx, int64_t batch, int64_t block, int64_t rank, const double* a_vt,
                       const double* b_u, const double* a_x, const double* b_x, double* g,
                       cudaStream_t s) {
  if (batch == 0) return LRB_OK;
  const int path = lowrank_path(block, rank, a_vt, b_u);
  if (path == 0) {
    LrProblem p;
    std::memset(&p, 0, sizeof(p));
    p.a_vt = a_vt;
    p.b_u = b_u;
    p.a_x = a_x;
    p.b_x = b_x;
    p.g = g;
    p.batch = batch;
    p.block = int(block);
    p.rank = int(rank);
    const int R = rank <= 8 ? 8 : rank <= 16 ? 16 : 32;
    const int G = 4, KB = R >= 32 ? 16 : 32;
    p.groups = (batch + G - 1) / G;
    const bool pair = (rank & 1) != 0;
    bool ok = encode3(&p.tmAV, a_vt, block, rank, batch, block, rank * block, KB + kPad, R, G) &&
              (pair ? encode3(&p.tmBU, b_u, 2 * rank, block / 2, batch, 2 * rank, block * rank,
                              2 * R + 4, KB / 2, G)
                    : encode3(&p.tmBU, b_u, rank, block, batch, rank, block * rank, R + kPad, KB, G));
    if (ok) {
      int64_t grid = 0;
      const int dev = ctx->device, sms = ctx->sm_count;
      cudaError_t e =
          pair ? (R == 8    ? launch_fast<8, true>(p, dev, sms, s, &grid)
                  : R == 16 ? launch_fast<16, true>(p, dev, sms, s, &grid)
                            : launch_fast<32, true>(p, dev, sms, s, &grid))
               : (R == 8    ? launch_fast<8, false>(p, dev, sms, s, &grid)
                  : R == 16 ? launch_fast<16, false>(p, dev, sms, s, &grid)
                            : launch_fast<32, false>(p, dev, sms, s, &grid));
      if (e != cudaSuccess) return cuda_fail(ctx, e, "lrb_lowrank_kernel launch");
      if (grid > 0) ctx->launches.fetch_add(1, std::memory_order_relaxed);
      return LRB_OK;
    }
  }
  if (path == 1 && lowrank_big_eligible(batch, block, rank, a_vt, b_u, a_x, b_x))
    return run_lowrank_big(ctx, batch, block, rank, a_vt, b_u, a_x, b_x, g, s);
  if (path == 1) {
    // C = A_Vt B_U, E = A_X C, G = E B_X as three row-major batched GEMMs
    // (the context workspace, not a stream-ordered allocation: inside a CUDA
    // graph an allocation becomes a memory node that is mapped per replay)
    double* scratch = nullptr;
    const size_t bytes = size_t(batch) * size_t(rank * rank) * 2 * sizeof(double);
    bool temp = false;
    lrb_status wst = acquire_workspace(ctx, bytes, s, reinterpret_cast<void**>(&scratch), &temp);
    if (wst) return wst;
    double* c = scratch;
    double* e = scratch + size_t(batch) * size_t(rank * rank);
    const int64_t rr = rank * rank;
    lrb_status st = run_strided_rowmajor(ctx, rank, rank, block, a_vt, rank * block, b_u,
                                         block * rank, c, rr, batch, s);
    if (!st) st = run_strided_rowmajor(ctx, rank, rank, rank, a_x, rr, c, rr, e, rr, batch, s);
    if (!st) st = run_strided_rowmajor(ctx, rank, rank, rank, e, rr, b_x, rr, g, rr, batch, s);
    release_workspace(ctx, s, scratch, temp);
    return st;
  }
  const size_t smem = size_t(2) * rank * rank * sizeof(double);
  if (smem > 200 * 1024)
    return fail(ctx, LRB_ERR_UNSUPPORTED, "lrb_lowrank_multiply: rank %lld too large", (long long)rank);
  if (smem > 48 * 1024)
    LRB_CUDA_TRY(ctx, cudaFuncSetAttribute(lrb_lowrank_simple_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t grid = std::min<int64_t>(batch, int64_t(ctx->sm_count) * 8);
  LRB_CUDA_TRY(ctx, launch_pdl(lrb_lowrank_simple_kernel, dim3(unsigned(grid)), dim3(128), smem,
                                s, a_vt, b_u, a_x, b_x, g, batch, int(block), int(rank)));
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
  return LRB_OK;
}

}  // namespace lrb

using namespace lrb;

static lrb_status validate_lowrank(lrb_ctx* ctx, const char* fn, int64_t batch, int64_t block,
                                   int64_t rank, const void* a_vt, const void* b_u, const void* a_x,
                                   const void* b_x, const void* g) {
  // LowRankBatch invariants (low_rank.hpp:123-133, validate :162-175)
  if (batch < 0) return fail(ctx, LRB_ERR_SHAPE, "%s: batch_size must be >= 0", fn);
  if (block < 1) return fail(ctx, LRB_ERR_SHAPE, "%s: block_size must be >= 1", fn);
  if (rank < 1) return fail(ctx, LRB_ERR_SHAPE, "%s: ranks must be >= 1", fn);
  if (block > INT32_MAX || rank > 4096)
    return fail(ctx, LRB_ERR_UNSUPPORTED, "%s: block or rank too large", fn);
  if (batch > 0 && (!a_vt || !b_u || !a_x || !b_x || !g))
    return fail(ctx, LRB_ERR_ARG, "%s: a role array is null", fn);
  return LRB_OK;
}

extern "C" lrb_status lrb_lowrank_multiply(lrb_ctx* ctx, int64_t batch, int64_t block,
                                           int64_t rank, const double* a_vt, const double* b_u,
                                           const double* a_x, const double* b_x, double* g,
                                           void* stream) {
  static const char* fn = "lrb_lowrank_multiply";
  lrb_status st = validate_lowrank(ctx, fn, batch, block, rank, a_vt, b_u, a_x, b_x, g);
  if (st) return st;
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "%s: null ctx", fn);
  st = bind(ctx);
  if (st) return st;
  return run_lowrank(ctx, batch, block, rank, a_vt, b_u, a_x, b_x, g,
                     static_cast<cudaStream_t>(stream));
}

extern "C" lrb_status lrb_lowrank_multiply_host(lrb_ctx* ctx, int64_t batch, int64_t block,
                                                int64_t rank, const double* a_vt,
                                                const double* b_u, const double* a_x,
                                                const double* b_x, double* g) {
  static const char* fn = "lrb_lowrank_multiply_host";
  lrb_status st = validate_lowrank(ctx, fn, batch, block, rank, a_vt, b_u, a_x, b_x, g);
  if (st) return st;
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "%s: null ctx", fn);
  if (batch == 0) return LRB_OK;
  st = bind(ctx);
  if (st) return st;
  // chunk the batch; H2D of the four roles, kernel, D2H of G per chunk on the
  // context's three pipeline streams
  const int64_t per_item = 2 * rank * block + 3 * rank * rank;  // doubles
  const int64_t target = (int64_t(128) << 20) / 8;
  const int64_t per_chunk = std::max<int64_t>(1, std::min<int64_t>(batch, target / per_item));
  const int64_t nchunks = (batch + per_chunk - 1) / per_chunk;
  const int lanes = int(std::min<int64_t>(lrb_ctx::kLanes, nchunks));
  const size_t need = size_t(per_item * per_chunk + 5 * 32) * 8;
  for (int l = 0; l < lanes; ++l) {
    if (ctx->lane_bytes[l] < need) {
      LRB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->lane_stream[l]));
      if (ctx->lane_buf[l]) cudaFree(ctx->lane_buf[l]);
      ctx->lane_buf[l] = nullptr;
      ctx->lane_bytes[l] = 0;
      LRB_CUDA_TRY(ctx, cudaMalloc(&ctx->lane_buf[l], need));
      ctx->lane_bytes[l] = need;
    }
  }
  auto r32 = [](int64_t x) { return (x + 31) / 32 * 32; };
  const int64_t rb = rank * block, rr = rank * rank;
  // pageable host buffers go through pinned staging (HostPipe)
  HostPipe pipe(ctx, lanes);
  const bool page_in = !host_pinned(a_vt) || !host_pinned(b_u) || !host_pinned(a_x) ||
                       !host_pinned(b_x);
  const bool page_out = !host_pinned(g);
  st = pipe.prepare(page_in ? size_t(per_item * per_chunk) * 8 + 4 * 256 : 0,
                    page_out ? size_t(rr * per_chunk) * 8 : 0);
  if (st) return st;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int l = int(c % lanes);
    cudaStream_t s = ctx->lane_stream[l];
    const int64_t i0 = c * per_chunk, n = std::min(per_chunk, batch - i0);
    double* dav = ctx->lane_buf[l];
    double* dbu = dav + r32(rb * per_chunk);
    double* dax = dbu + r32(rb * per_chunk);
    double* dbx = dax + r32(rr * per_chunk);
    double* dg = dbx + r32(rr * per_chunk);
    if ((st = pipe.begin(l))) return st;
    if ((st = pipe.h2d(l, dav, a_vt + i0 * rb, size_t(n * rb) * 8))) return st;
    if ((st = pipe.h2d(l, dbu, b_u + i0 * rb, size_t(n * rb) * 8))) return st;
    if ((st = pipe.h2d(l, dax, a_x + i0 * rr, size_t(n * rr) * 8))) return st;
    if ((st = pipe.h2d(l, dbx, b_x + i0 * rr, size_t(n * rr) * 8))) return st;
    if ((st = pipe.inputs_done(l))) return st;
    st = run_lowrank(ctx, n, block, rank, dav, dbu, dax, dbx, dg, s);
    if (st) return st;
    if ((st = pipe.d2h(l, g + i0 * rr, dg, size_t(n * rr) * 8))) return st;
    if ((st = pipe.outputs_done(l))) return st;
  }
  return pipe.finish();
}

extern "C" double lrb_lowrank_flops_per_item(int64_t rank, int64_t block) {
  // the reference's accounting, flops_per_item (low_rank.hpp:66-68)
  return 4.0 * double(rank) * rank * rank + 2.0 * double(rank) * rank * block;
}

// ------------------------------------------------------ low-rank expansion
namespace lrb {
lrb_status run_strided_rowmajor_beta(lrb_ctx* ctx, int64_t m, int64_t n, int64_t k,
                                     const double* A, int64_t lda, int64_t sA, const double* B,
                                     int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC,
                                     int64_t batch, int beta_one, cudaStream_t stream);
bool launch_expand_stream(lrb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t r,
                          const double* u, int64_t su, const double* x, int64_t sx,
                          const double* vt, int64_t svt, double* out, int64_t ldo, int64_t so,
                          cudaStream_t s, lrb_status* st);
}

// out_i = (U_i X_i) Vt_i, the reference's per-tile expansion (blr.hpp:75-78):
// UX (m x r, K = r) into the context workspace, then UX Vt (m x n, K = r) —
// the cfg2 shape (U V^T with an r x r core), q64 tiles.
extern "C" lrb_status lrb_lowrank_expand(lrb_ctx* ctx, int64_t batch, int64_t m, int64_t n,
                                         int64_t rank, const double* u, int64_t su,
                                         const double* x, int64_t sx, const double* vt,
                                         int64_t svt, double* out, int64_t ldo, int64_t so,
                                         void* stream) {
  static const char* fn = "lrb_lowrank_expand";
  // LowRankOperand invariants and messages (low_rank.hpp:56-61)
  if (rank < 1) return fail(ctx, LRB_ERR_SHAPE, "LowRankOperand: rank must be >= 1");
  if (m < rank || n < rank)
    return fail(ctx, LRB_ERR_SHAPE,
                "LowRankOperand: need m >= rank and n >= rank, got (%lld, %lld, %lld)",
                (long long)m, (long long)n, (long long)rank);
  if (batch < 0) return fail(ctx, LRB_ERR_SHAPE, "%s: batch must be >= 0", fn);
  if (ldo < n)
    return fail(ctx, LRB_ERR_SHAPE, "%s: ldo is %lld but out is %lldx%lld", fn, (long long)ldo,
                (long long)m, (long long)n);
  if (su < 0 || sx < 0 || svt < 0)
    return fail(ctx, LRB_ERR_SHAPE, "%s: input strides must be >= 0", fn);
  if (batch > 1 && so < (m - 1) * ldo + n)
    return fail(ctx, LRB_ERR_SHAPE, "%s: stride %lld < %lld: output items would overlap", fn,
                (long long)so, (long long)((m - 1) * ldo + n));
  if (!u || !x || !vt || !out) return fail(ctx, LRB_ERR_ARG, "%s: null operand", fn);
  if (!ctx) return fail(nullptr, LRB_ERR_ARG, "%s: null ctx", fn);
  if (batch == 0) return LRB_OK;
  lrb_status st = bind(ctx);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // rank 8 / 16 with 64-row, 256-column items: one write-streaming launch, UX
  // kept on chip (lrb_blr_recon.cu); LRB_EXPAND_STREAM=0 keeps the two GEMMs
  const char* es = std::getenv("LRB_EXPAND_STREAM");
  if (!(es && es[0] == '0') &&
      lrb::launch_expand_stream(ctx, batch, m, n, rank, u, su, x, sx, vt, svt, out, ldo, so, s, &st))
    return st;
  double* ux = nullptr;
  bool temp = false;
  const size_t bytes = size_t(batch) * size_t(m * rank) * sizeof(double);
  st = acquire_workspace(ctx, bytes, s, reinterpret_cast<void**>(&ux), &temp);
  if (st) return st;
  st = run_strided_rowmajor_beta(ctx, m, rank, rank, u, rank, su, x, rank, sx, ux, rank, m * rank,
                                 batch, 0, s);
  if (!st)
    st = run_strided_rowmajor_beta(ctx, m, n, rank, ux, rank, m * rank, vt, n, svt, out, ldo, so,
                                   batch, 0, s);
  release_workspace(ctx, s, ux, temp);
  return st;
}
