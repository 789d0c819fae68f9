// lrb_dispatch.cuh — variant traits generated from the variant table, and the
// per-variant launch entry (explicitly instantiated once per variant in
// lrb_gemm_v*.cu so the 9 x 4 x 2 kernels compile in parallel units).
#pragma once

#include "lrb_gemm.cuh"
#include "lrb_variants.h"

namespace lrb {

template <int ID>
struct VariantTraits;

#define LRB_X(id, nm, WARPS_I, WARPS_J, WI, WJ, KB, ST, MINB)                        \
  template <>                                                                        \
  struct VariantTraits<id> {                                                         \
    template <bool AT, bool BT, bool TMA>                                            \
    using Cfg = GemmCfg<WARPS_I, WARPS_J, WI, WJ, KB, ST, MINB, AT, BT, TMA>;        \
    static constexpr const char* name = #nm;                                         \
  };
LRB_VARIANT_LIST(LRB_X)
#undef LRB_X

// a_t / b_t: op flags of the column-major view; tma: operands loaded through
// tensor maps (else per-segment bulk copies); exactly one of sp / pp non-null.
template <int ID>
cudaError_t launch_variant(int a_t, int b_t, int tma, const StridedProblem* sp,
                           const PtrProblem* pp, int beta_one, int device, int sm_count,
                           cudaStream_t stream, LaunchInfo* info) {
  using VT = VariantTraits<ID>;
#define LRB_CASE(AT, BT, TM)                                                                   \
  if (a_t == AT && b_t == BT && (tma != 0) == TM) {                                            \
    using C = typename VT::template Cfg<AT, BT, TM>;                                           \
    return sp ? launch_gemm<C>(*sp, beta_one, device, sm_count, stream, info)                  \
              : launch_gemm<C>(*pp, beta_one, device, sm_count, stream, info);                 \
  }
  LRB_CASE(0, 0, true)
  LRB_CASE(0, 1, true)
  LRB_CASE(1, 0, true)
  LRB_CASE(1, 1, true)
  LRB_CASE(0, 0, false)
  LRB_CASE(0, 1, false)
  LRB_CASE(1, 0, false)
  LRB_CASE(1, 1, false)
#undef LRB_CASE
  return cudaErrorInvalidValue;
}

using LaunchFn = cudaError_t (*)(int, int, int, const StridedProblem*, const PtrProblem*, int, int,
                                 int, cudaStream_t, LaunchInfo*);

#define LRB_X(id, ...)                                                                         \
  extern template cudaError_t launch_variant<id>(int, int, int, const StridedProblem*,         \
                                                 const PtrProblem*, int, int, int, cudaStream_t, \
                                                 LaunchInfo*);
LRB_VARIANT_LIST(LRB_X)
#undef LRB_X

}  // namespace lrb
