"""ctypes binding of the C-ABI in include/lrb.h (liblrb.so, built in-tree).

The shared library is the product: there is no Python or CPU fallback. If the
in-tree ``liblrb.so`` is missing, importing this module raises. The library is
mapped into the process on the first call through ``lib`` (not at import), so
processes that only use the host-side workload definitions (bench.py's CPU
reference arm) never load it.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblrb.so")

# status codes (include/lrb.h)
LRB_OK = 0
LRB_ERR_SHAPE = 1
LRB_ERR_CAPACITY = 2
LRB_ERR_ARG = 3
LRB_ERR_CUDA = 4
LRB_ERR_UNSUPPORTED = 5
LRB_ERR_NO_DEVICE = 6
LRB_ERR_IO = 7
LRB_ERR_PARSE = 8

i64 = C.c_int64
u64 = C.c_uint64
u32 = C.c_uint32
dbl = C.c_double
vp = C.c_void_p
P = C.POINTER


class lrb_selection(C.Structure):
    _fields_ = [
        ("variant", C.c_int),
        ("tile_m", C.c_int),
        ("tile_n", C.c_int),
        ("tile_k", C.c_int),
        ("stages", C.c_int),
        ("threads", C.c_int),
        ("ctas_per_sm", C.c_int),
        ("tiles", i64),
        ("grid", i64),
        ("intensity", dbl),
        ("fp64_bound", C.c_int),
        ("name", C.c_char * 24),
    ]


# name -> (restype, argtypes); every symbol include/lrb.h declares
SIGNATURES = {
    "lrb_create": (C.c_int, [C.c_int, P(vp)]),
    "lrb_destroy": (C.c_int, [vp]),
    "lrb_last_error": (C.c_char_p, [vp]),
    "lrb_version": (C.c_char_p, []),
    "lrb_device_count": (C.c_int, []),
    "lrb_device_name": (C.c_int, [C.c_int, C.c_char_p, C.c_size_t]),
    "lrb_ctx_device": (C.c_int, [vp]),
    "lrb_ctx_sm_count": (C.c_int, [vp]),
    "lrb_launch_count": (u64, [vp]),
    "lrb_last_variant": (C.c_int, [vp]),
    "lrb_malloc": (C.c_int, [vp, C.c_size_t, P(vp)]),
    "lrb_free": (C.c_int, [vp, vp]),
    "lrb_host_alloc": (C.c_int, [vp, C.c_size_t, P(vp)]),
    "lrb_host_free": (C.c_int, [vp, vp]),
    "lrb_memcpy_h2d": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "lrb_memcpy_d2h": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "lrb_memset": (C.c_int, [vp, vp, C.c_int, C.c_size_t]),
    "lrb_stream_create": (C.c_int, [vp, P(vp)]),
    "lrb_stream_destroy": (C.c_int, [vp, vp]),
    "lrb_stream_sync": (C.c_int, [vp, vp]),
    "lrb_device_sync": (C.c_int, [vp]),
    "lrb_mem_info": (C.c_int, [vp, P(C.c_size_t), P(C.c_size_t)]),
    "lrb_event_create": (C.c_int, [vp, P(vp)]),
    "lrb_event_destroy": (C.c_int, [vp, vp]),
    "lrb_event_record": (C.c_int, [vp, vp, vp]),
    "lrb_event_elapsed_ms": (C.c_int, [vp, vp, vp, P(C.c_float)]),
    "lrb_l2_flush": (C.c_int, [vp, vp]),
    "lrb_l2_evict": (C.c_int, [vp, vp]),
    "lrb_dgemm_strided_batched": (
        C.c_int,
        [vp, C.c_char, C.c_char, C.c_char, i64, i64, i64, dbl, vp, i64, i64, vp, i64, i64, vp, i64,
         i64, i64, vp],
    ),
    "lrb_ptr_plan_create": (
        C.c_int,
        [vp, C.c_char, C.c_char, C.c_char, i64, P(i64), P(i64), P(i64), P(vp), P(i64), P(vp),
         P(i64), P(vp), P(i64), dbl, P(vp)],
    ),
    "lrb_ptr_plan_execute": (C.c_int, [vp, vp, vp]),
    "lrb_ptr_plan_destroy": (C.c_int, [vp, vp]),
    "lrb_ptr_plan_launches": (C.c_int, [vp]),
    "lrb_dgemm_ptr_batched": (
        C.c_int,
        [vp, C.c_char, C.c_char, C.c_char, i64, P(i64), P(i64), P(i64), P(vp), P(i64), P(vp),
         P(i64), P(vp), P(i64), dbl, vp],
    ),
    "lrb_gemm_naive_raw": (
        C.c_int, [vp, vp, vp, vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, P(u64)]
    ),
    "lrb_dgemm_strided_batched_host": (
        C.c_int,
        [vp, C.c_char, C.c_char, C.c_char, i64, i64, i64, dbl, vp, i64, i64, vp, i64, i64, vp, i64,
         i64, i64],
    ),
    "lrb_dgemm_ptr_batched_device": (
        C.c_int,
        [vp, C.c_char, C.c_char, C.c_char, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, dbl, vp, vp],
    ),
    "lrb_dgemm_ptr_batched_host": (
        C.c_int,
        [vp, C.c_char, C.c_char, C.c_char, i64, P(i64), P(i64), P(i64), P(vp), P(i64), P(vp),
         P(i64), P(vp), P(i64), dbl],
    ),
    "lrb_lowrank_multiply": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp]),
    "lrb_lowrank_multiply_host": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp]),
    "lrb_lowrank_expand": (C.c_int, [vp, i64, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                                     i64, vp]),
    "lrb_lowrank_flops_per_item": (dbl, [i64, i64]),
    "lrb_batch_file_header": (C.c_int, [C.c_char_p, P(i64)]),
    "lrb_batch_file_load": (C.c_int, [vp, C.c_char_p, vp, vp, vp, vp, C.c_int]),
    "lrb_batch_file_save": (C.c_int, [vp, C.c_char_p, i64, i64, i64, i64, vp, vp, vp, vp, C.c_int]),
    "lrb_blr_create": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, P(vp)]),
    "lrb_blr_matvec": (C.c_int, [vp, vp, vp, i64, vp]),
    "lrb_blr_matvec_device": (C.c_int, [vp, vp, vp, i64, vp, vp]),
    "lrb_blr_destroy": (C.c_int, [vp, vp]),
    "lrb_blr_reconstruct_dense": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "lrb_graph_begin": (C.c_int, [vp, vp]),
    "lrb_graph_end": (C.c_int, [vp, vp, P(vp)]),
    "lrb_graph_launch": (C.c_int, [vp, vp, vp]),
    "lrb_graph_destroy": (C.c_int, [vp, vp]),
    "lrb_graph_launches": (u64, [vp]),
    "lrb_select": (
        C.c_int, [vp, C.c_char, C.c_char, C.c_char, i64, i64, i64, i64, P(lrb_selection)]
    ),
    "lrb_variant_count": (C.c_int, []),
    "lrb_variant_name": (C.c_char_p, [C.c_int]),
    "lrb_variant_from_name": (C.c_int, [C.c_char_p]),
    "lrb_set_variant_override": (C.c_int, [vp, C.c_int]),
    "lrb_set_loader_override": (C.c_int, [vp, C.c_int]),
    "lrb_shard_plan": (C.c_int, [i64, P(dbl), C.c_int, P(i64)]),
    "lrb_item_flops": (dbl, [i64, i64, i64]),
    "lrb_item_bytes": (dbl, [i64, i64, i64, dbl]),
    "lrb_fill_uniform": (C.c_int, [vp, vp, i64, i64, i64, i64, i64, u64, u32, i64, vp]),
    "lrb_fill_uniform_ptr": (C.c_int, [vp, P(vp), P(i64), P(i64), P(i64), i64, u64, u32, i64, vp]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
            "there is no CPU fallback"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """``liblrb.so`` bound on first use (every attribute is a C-ABI symbol)"""

    _cdll = None

    def __getattr__(self, name):
        if _LazyLib._cdll is None:
            _LazyLib._cdll = _load()
        return getattr(_LazyLib._cdll, name)

    @staticmethod
    def loaded() -> bool:
        return _LazyLib._cdll is not None


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` (or "
                      "__graft_entry__.build()); there is no CPU fallback")
lib = _LazyLib()
