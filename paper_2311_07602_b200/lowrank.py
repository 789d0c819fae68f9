"""The paper's batched low-rank product on the GPU, reference-shaped.

Mirrors the reference's LowRankBatch (proj/include/lrbatch/low_rank.hpp:109-176)
and its drivers fused_multiply / packed_multiply (kernels.hpp:131-161,
243-349): ``G_i = A_X_i (A_Vt_i B_U_i) B_X_i`` for every item, all matrices
row-major, each role packed contiguously. Both drivers run the same B200 kernel
(lrb_lowrank_multiply): one warp per item, TMA-fed DMMA for A_Vt B_U, the two
small products from registers, G stored once. ``plan``/``workers`` arguments are
accepted for signature compatibility; the GPU needs neither.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import workloads as W
from .lrbatch import ArgError, Context, ShapeError, _check, default_context, lib


def flops_per_item(rank: int, block_size: int) -> int:
    """4 r^3 + 2 r^2 b (reference low_rank.hpp:66-68)"""
    return 4 * rank * rank * rank + 2 * rank * rank * block_size


class LowRankBatch:
    """Five contiguous role arrays, item i of a role at i*rows*cols (row-major)."""

    def __init__(self, batch_size: int, block_size: int, rank_a: int, rank_b: int):
        if batch_size < 1:
            raise ShapeError("LowRankBatch: batch_size must be >= 1")
        if block_size < 1:
            raise ShapeError("LowRankBatch: block_size must be >= 1")
        if rank_a < 1 or rank_b < 1:
            raise ShapeError("LowRankBatch: ranks must be >= 1")
        self.batch_size, self.block_size = batch_size, block_size
        self.rank_a, self.rank_b = rank_a, rank_b
        self.a_vt_batch = np.zeros(batch_size * rank_a * block_size)
        self.b_u_batch = np.zeros(batch_size * block_size * rank_b)
        self.a_x_batch = np.zeros(batch_size * rank_a * rank_a)
        self.b_x_batch = np.zeros(batch_size * rank_b * rank_b)
        self.g_xy_batch = np.zeros(batch_size * rank_a * rank_b)
        self.seed: Optional[int] = None

    @staticmethod
    def random(batch: int, block: int, rank: int, seed: int) -> "LowRankBatch":
        """Seeded operands. The reference draws N(0,1) from one sequential
        mt19937_64 stream (low_rank.hpp:135-145); this build draws
        uniform[-1,1) from the counter RNG (include/lrb_rng.h, roles 0..3) so any
        item regenerates independently on host or device."""
        b = LowRankBatch(batch, block, rank, rank)
        for role, arr in enumerate((b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)):
            key = W.stream_key(seed, role)
            per = arr.size // batch
            idx = np.arange(per, dtype=np.uint64)
            for it in range(batch):
                arr[it * per:(it + 1) * per] = _uniform_vec(key, it, idx)
        b.seed = seed
        return b

    def a_vt(self, item):
        n = self.rank_a * self.block_size
        return self.a_vt_batch[item * n:(item + 1) * n].reshape(self.rank_a, self.block_size)

    def b_u(self, item):
        n = self.block_size * self.rank_b
        return self.b_u_batch[item * n:(item + 1) * n].reshape(self.block_size, self.rank_b)

    def a_x(self, item):
        n = self.rank_a * self.rank_a
        return self.a_x_batch[item * n:(item + 1) * n].reshape(self.rank_a, self.rank_a)

    def b_x(self, item):
        n = self.rank_b * self.rank_b
        return self.b_x_batch[item * n:(item + 1) * n].reshape(self.rank_b, self.rank_b)

    def g_xy(self, item):
        n = self.rank_a * self.rank_b
        return self.g_xy_batch[item * n:(item + 1) * n].reshape(self.rank_a, self.rank_b)

    def zero_results(self) -> None:
        self.g_xy_batch[:] = 0.0

    def validate(self) -> None:
        """low_rank.hpp:162-175"""
        b, k, ra, rb = self.batch_size, self.block_size, self.rank_a, self.rank_b
        if not (b >= 1 and k >= 1 and ra >= 1 and rb >= 1):
            raise ShapeError("LowRankBatch: degenerate dimensions")
        for name, arr, want in (("a_vt_batch", self.a_vt_batch, b * ra * k),
                                ("b_u_batch", self.b_u_batch, b * k * rb),
                                ("a_x_batch", self.a_x_batch, b * ra * ra),
                                ("b_x_batch", self.b_x_batch, b * rb * rb),
                                ("g_xy_batch", self.g_xy_batch, b * ra * rb)):
            if arr.size != want:
                raise ShapeError(f"LowRankBatch: {name} length mismatch")
            if arr.dtype != np.float64 or not arr.flags.c_contiguous:
                raise ArgError(f"LowRankBatch: {name} must be contiguous float64")


def _uniform_vec(key: int, item: int, idx: np.ndarray) -> np.ndarray:
    """vectorised include/lrb_rng.h lrb_uniform for one item"""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        z = (np.uint64(key) + ((np.uint64(item) << np.uint64(32)) | idx) *
             np.uint64(0x9E3779B97F4A7C15)) & M
        z ^= z >> np.uint64(30)
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z = z * np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 4503599627370496.0) - 1.0


def _run(batch: LowRankBatch, who: str, ctx: Optional[Context]) -> None:
    batch.validate()
    if batch.rank_a != batch.rank_b:
        raise ShapeError(f"{who}: rank_a must equal rank_b (got {batch.rank_a} and "
                         f"{batch.rank_b})")
    ctx = ctx or default_context()
    _check(lib.lrb_lowrank_multiply_host(
        ctx._h, batch.batch_size, batch.block_size, batch.rank_a,
        batch.a_vt_batch.ctypes.data, batch.b_u_batch.ctypes.data, batch.a_x_batch.ctypes.data,
        batch.b_x_batch.ctypes.data, batch.g_xy_batch.ctypes.data), ctx._h)


def fused_multiply(batch: LowRankBatch, ctx: Optional[Context] = None) -> None:
    """Drop-in for lrbatch::fused_multiply (kernels.hpp:131-161), on the GPU."""
    _run(batch, "fused_multiply", ctx)


def packed_multiply(batch: LowRankBatch, plan=None, workers: int = 1, stats=None,
                    ctx: Optional[Context] = None) -> None:
    """Drop-in for lrbatch::packed_multiply (kernels.hpp:243-349), on the GPU.
    ``plan`` and ``workers`` (CPU cache blocking and thread fan-out) do not apply.
    ``stats``, when a dict, receives g_entry_stores = batch * rank_a * rank_b
    (every G entry is stored exactly once, like the register-tile path)."""
    _run(batch, "packed_multiply", ctx)
    if isinstance(stats, dict):
        stats["g_entry_stores"] = batch.batch_size * batch.rank_a * batch.rank_b


def lowrank_multiply_device(ctx: Context, batch: int, block: int, rank: int, a_vt, b_u, a_x, b_x,
                            g, stream=None) -> None:
    """Device-pointer form (lrb_lowrank_multiply)."""
    from .lrbatch import _ptr

    _check(lib.lrb_lowrank_multiply(ctx._h, batch, block, rank, _ptr(a_vt), _ptr(b_u), _ptr(a_x),
                                    _ptr(b_x), _ptr(g), stream.handle if stream else None),
           ctx._h)


# ------------------------------------------------------ LRBATCH1 batch files
def save_batch(batch: LowRankBatch, path: str) -> None:
    """lrbatch::save_batch (batch_io.hpp:29-47)"""
    import ctypes as C

    batch.validate()
    _check(lib.lrb_batch_file_save(None, path.encode(), batch.batch_size, batch.block_size,
                                   batch.rank_a, batch.rank_b, batch.a_vt_batch.ctypes.data,
                                   batch.b_u_batch.ctypes.data, batch.a_x_batch.ctypes.data,
                                   batch.b_x_batch.ctypes.data, 0), None)


def batch_file_header(path: str):
    import ctypes as C

    hdr = (C.c_int64 * 4)()
    _check(lib.lrb_batch_file_header(path.encode(), hdr), None)
    return tuple(int(x) for x in hdr)


def load_batch(path: str) -> LowRankBatch:
    """lrbatch::load_batch (batch_io.hpp:49-77): zeroed results"""
    n, block, ra, rb = batch_file_header(path)
    out = LowRankBatch(n, block, ra, rb)
    _check(lib.lrb_batch_file_load(None, path.encode(), out.a_vt_batch.ctypes.data,
                                   out.b_u_batch.ctypes.data, out.a_x_batch.ctypes.data,
                                   out.b_x_batch.ctypes.data, 0), None)
    return out


def load_batch_device(ctx: Context, path: str):
    """Stream a batch file into device memory: returns (header, [a_vt, b_u,
    a_x, b_x] DeviceBuffers, g DeviceBuffer) ready for lowrank_multiply_device."""
    n, block, ra, rb = batch_file_header(path)
    bufs = [ctx.empty(n * ra * block), ctx.empty(n * block * rb), ctx.empty(n * ra * ra),
            ctx.empty(n * rb * rb)]
    _check(lib.lrb_batch_file_load(ctx._h, path.encode(), *[b.ptr for b in bufs], 1), ctx._h)
    return (n, block, ra, rb), bufs, ctx.empty(n * ra * rb)
