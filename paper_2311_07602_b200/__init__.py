"""lrb-b200: B200-native batched FP64 GEMM for low-rank / BLR blocks.

The hot path of arXiv 2311.07602's reference (lrbatch's ``gemm_naive_raw``
over batches, proj/include/lrbatch/dense.hpp:43-56) as hand-written sm_100a
CUDA behind the C-ABI in ``include/lrb.h``. ``lrbatch`` is the
reference-shaped Python mirror of that ABI.
"""
from .lrbatch import (  # noqa: F401
    ArgError,
    CapacityError,
    Context,
    CudaError,
    DenseBlock,
    DeviceBuffer,
    IoError,
    LrbError,
    ParseError,
    NoDeviceError,
    PinnedBuffer,
    PtrPlan,
    ShapeError,
    UnsupportedError,
    default_context,
    dense_gemm_naive,
    device_count,
    gemm_naive_raw,
    item_bytes,
    item_flops,
    select,
    shard_plan,
    variant_from_name,
    variant_names,
    version,
)

# operand roles of the synthetic-input generator (include/lrb_rng.h)
ROLE_A, ROLE_B, ROLE_C, ROLE_SHAPE_B, ROLE_SHAPE_R = 0, 1, 2, 3, 4
