// Instantiation unit for kernel variant 24 of the table in lrb_variants.h.
#include "lrb_dispatch.cuh"
namespace lrb {
template cudaError_t launch_variant<24>(int, int, int, const StridedProblem*, const PtrProblem*,
                                        int, int, int, cudaStream_t, LaunchInfo*);
}  // namespace lrb
