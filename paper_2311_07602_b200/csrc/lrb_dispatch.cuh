// lrb_dispatch.cuh — variant traits generated from the variant table, and the
// per-variant launch entry (explicitly instantiated once per variant in
// lrb_gemm_v*.cu so the 9 x 4 x 2 kernels compile in parallel units).
#pragma once

#include <type_traits>

#include "lrb_gemm.cuh"
#include "lrb_variants.h"

namespace lrb {

template <int ID>
struct VariantTraits;

// Variants whose TMA instantiations run a producer warp (ProdCfg): the
// 4-warp tile shapes, where the fifth warp still leaves >= 128 registers per
// thread. Measured against the all-computing-warps form on one box
// (DESIGN.md 4.1): r = 32 class 0.79-0.83 -> 0.90-0.94 of FP64 peak, r = 16
// rows 0.97-1.05 -> 1.05-1.09 of HBM, row-major short-wide rows +2-14%, the
// BLR matvec +7-13%; n48 / n56 as four 32 x 48 / 32 x 56 warps with the
// producer beat their former 8-warp shapes by 2.6% / 4-4.5%. The 8-warp
// shapes (n64, n64s4, sq, m64) were neutral to -2.4%, s96 -8% and q64 with
// its TMA-store epilogue -9%: those keep the release-counter form.
template <int ID>
struct VariantProd {
  static constexpr bool value =
      ID == LRB_V_N8 || ID == LRB_V_N16 || ID == LRB_V_N24 || ID == LRB_V_N32 ||
      ID == LRB_V_N40 || ID == LRB_V_N48 || ID == LRB_V_N56 || ID == LRB_V_M8 ||
      ID == LRB_V_M16 || ID == LRB_V_M32 ||
      ID == LRB_V_N16T || ID == LRB_V_N16H || ID == LRB_V_M8T || ID == LRB_V_M16T ||
      ID == LRB_V_T64 || ID == LRB_V_M16K64 || ID == LRB_V_M8K64 || ID == LRB_V_Q64P ||
      ID == LRB_V_Q64Q;
};

// variants that run a producer warpgroup with setmaxnreg (ProdWgCfg): s96,
// whose 48 x 48 warp tiles need ~200 registers per thread
template <int ID>
struct VariantProdWg {
  static constexpr bool value = ID == LRB_V_S96;
};

#define LRB_X(id, nm, WARPS_I, WARPS_J, WI, WJ, KB, ST, MINB)                        \
  template <>                                                                        \
  struct VariantTraits<id> {                                                         \
    template <bool AT, bool BT, bool TMA>                                            \
    using Base = GemmCfg<WARPS_I, WARPS_J, WI, WJ, KB, ST, MINB, AT, BT, TMA>;       \
    template <bool AT, bool BT, bool TMA>                                            \
    using Cfg = std::conditional_t<                                                  \
        VariantProdWg<id>::value && TMA, ProdWgCfg<Base<AT, BT, TMA>, 40, 216>,      \
        std::conditional_t<VariantProd<id>::value && TMA, ProdCfg<Base<AT, BT, TMA>>, \
                           Base<AT, BT, TMA>>>;                                      \
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
