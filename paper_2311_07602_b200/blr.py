"""BLR multi-RHS matvec on the GPU, reference-shaped.

Mirrors the reference's BlrMatrix / blr_matvec (proj/include/lrbatch/blr.hpp:
15-175): a weakly admissible block low-rank matrix (dense diagonal tiles,
U X Vt off-diagonal tiles over a uniform grid) times a block of right-hand
sides. The matrix is uploaded once (lrb_blr_create, device layout built for
the four batched launches of lrb_blr_matvec); every product keeps the
reference's chain order.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import workloads as W
from .lowrank import _uniform_vec
from .lrbatch import Context, DenseBlock, ShapeError, _check, default_context, lib


class LowRankOperand:
    """U (m x rank) X (rank x rank) Vt (rank x n), row-major (low_rank.hpp:16-63)."""

    def __init__(self, m: int, n: int, rank: int, u=None, x=None, vt=None):
        if rank < 1:
            raise ShapeError("LowRankOperand: rank must be >= 1")
        if m < rank or n < rank:
            raise ShapeError(f"LowRankOperand: need m >= rank and n >= rank, got ({m}, {n}, {rank})")
        self.m, self.n, self.rank = m, n, rank
        self.u = np.zeros(m * rank) if u is None else np.ascontiguousarray(u, dtype=np.float64)
        self.x = np.zeros(rank * rank) if x is None else np.ascontiguousarray(x, dtype=np.float64)
        self.vt = np.zeros(rank * n) if vt is None else np.ascontiguousarray(vt, dtype=np.float64)


class BlrMatrix:
    """n = tiles * block_size; diagonal: tiles DenseBlocks; off_diagonal:
    tiles*(tiles-1) LowRankOperands, row-major over (i, j != i) (blr.hpp:15-87)."""

    def __init__(self, n: int, block_size: int, rank: int):
        if not (block_size >= 1 and n >= block_size):
            raise ShapeError("BlrMatrix: bad block size")
        if n % block_size:
            raise ShapeError(f"BlrMatrix: n = {n} is not a multiple of block_size {block_size}")
        if not (1 <= rank <= block_size):
            raise ShapeError("BlrMatrix: rank must be in [1, block]")
        self.n, self.block_size, self.rank = n, block_size, rank
        self.tiles = n // block_size
        self.diagonal: List[DenseBlock] = []
        self.off_diagonal: List[LowRankOperand] = []
        self._dev = None  # (ctx, handle) of the uploaded copy

    def off_index(self, i: int, j: int) -> int:
        return i * (self.tiles - 1) + (j if j < i else j - 1)

    def off_tile(self, i: int, j: int) -> LowRankOperand:
        return self.off_diagonal[self.off_index(i, j)]

    @staticmethod
    def random(n: int, block_size: int, rank: int, seed: int) -> "BlrMatrix":
        """Seeded tiles from the counter RNG (uniform[-1,1)); the reference
        draws N(0,1) from one sequential stream (blr.hpp:40-57)."""
        m = BlrMatrix(n, block_size, rank)
        b, r = block_size, rank
        for i in range(m.tiles):
            d = _uniform_vec(W.stream_key(seed, 10), i, np.arange(b * b, dtype=np.uint64))
            m.diagonal.append(DenseBlock(b, b, d))
        o = 0
        for i in range(m.tiles):
            for j in range(m.tiles):
                if i == j:
                    continue
                u = _uniform_vec(W.stream_key(seed, 11), o, np.arange(b * r, dtype=np.uint64))
                x = _uniform_vec(W.stream_key(seed, 12), o, np.arange(r * r, dtype=np.uint64))
                vt = _uniform_vec(W.stream_key(seed, 13), o, np.arange(r * b, dtype=np.uint64))
                m.off_diagonal.append(LowRankOperand(b, b, r, u, x, vt))
                o += 1
        return m

    def packed_arrays(self):
        """(diag, u, x, vt) concatenated in the reference order"""
        cat = lambda xs: np.ascontiguousarray(np.concatenate(xs)) if xs else np.zeros(1)  # noqa
        return (cat([d.data for d in self.diagonal]), cat([t.u for t in self.off_diagonal]),
                cat([t.x for t in self.off_diagonal]), cat([t.vt for t in self.off_diagonal]))

    def invalidate(self) -> None:
        """drop the device copy (call after editing tiles)"""
        if self._dev is not None:
            ctx, h = self._dev
            lib.lrb_blr_destroy(ctx._h, h)
        self._dev = None

    def device_handle(self, ctx: Context) -> int:
        if self._dev is not None and self._dev[0] is ctx:
            return self._dev[1]
        self.invalidate()
        if len(self.diagonal) != self.tiles or len(self.off_diagonal) != self.tiles * (self.tiles - 1):
            raise ShapeError("BlrMatrix: tiles are not populated")
        diag, u, x, vt = self.packed_arrays()
        h = C.c_void_p()
        _check(lib.lrb_blr_create(ctx._h, self.n, self.block_size, self.rank, diag.ctypes.data,
                                  u.ctypes.data, x.ctypes.data, vt.ctypes.data, C.byref(h)),
               ctx._h)
        self._dev = (ctx, h.value)
        return h.value

    def reconstruct_dense(self, ctx: Optional[Context] = None) -> DenseBlock:
        """Exact dense n x n assembly (BlrMatrix::reconstruct_dense,
        blr.hpp:62-86) on the GPU: diagonal tiles copied, off-diagonal tiles
        expanded as (U X) Vt in the reference's order."""
        ctx = ctx or default_context()
        h = self.device_handle(ctx)
        out = DenseBlock(self.n, self.n)
        _check(lib.lrb_blr_reconstruct_dense(ctx._h, h, out.data.ctypes.data, 0, None), ctx._h)
        return out

    def reconstruct_dense_device(self, ctx: Context, out, stream=None) -> None:
        """device form: `out` is a DeviceBuffer of n*n doubles (asynchronous)"""
        from .lrbatch import _ptr

        h = self.device_handle(ctx)
        _check(lib.lrb_blr_reconstruct_dense(ctx._h, h, _ptr(out), 1,
                                             stream.handle if stream else None), ctx._h)

    def __del__(self):
        try:
            self.invalidate()
        except Exception:
            pass


def blr_matvec(m: BlrMatrix, rhs: DenseBlock, plan=None, workers: int = 1,
               ctx: Optional[Context] = None) -> DenseBlock:
    """y = M rhs (blr_matvec, blr.hpp:141-175) on the GPU; plan/workers do not apply."""
    if rhs.rows != m.n:
        raise ShapeError(f"blr_matvec: rhs has {rhs.rows} rows, matrix has dimension {m.n}")
    ctx = ctx or default_context()
    h = m.device_handle(ctx)
    y = DenseBlock(m.n, rhs.cols)
    _check(lib.lrb_blr_matvec(ctx._h, h, rhs.data.ctypes.data, rhs.cols, y.data.ctypes.data),
           ctx._h)
    return y


def lowrank_expand(u, x, vt, batch: int, m: int, n: int, rank: int,
                   ctx: Optional[Context] = None) -> np.ndarray:
    """out_i = (U_i X_i) Vt_i for a uniform batch of LowRankOperands held as
    contiguous row-major host arrays (the per-tile expansion of
    reconstruct_dense, blr.hpp:75-78), computed on the GPU; returns
    batch * m * n doubles."""
    ctx = ctx or default_context()
    du, dx, dvt = ctx.to_device(u), ctx.to_device(x), ctx.to_device(vt)
    dout = ctx.empty(max(1, batch * m * n))
    lowrank_expand_device(ctx, batch, m, n, rank, du, dx, dvt, dout)
    ctx.synchronize()
    return dout.download()[: batch * m * n]


def lowrank_expand_device(ctx: Context, batch: int, m: int, n: int, rank: int, u, x, vt, out,
                          su: Optional[int] = None, sx: Optional[int] = None,
                          svt: Optional[int] = None, ldo: Optional[int] = None,
                          so: Optional[int] = None, stream=None) -> None:
    """device form of lrb_lowrank_expand (strides default to packed items)"""
    from .lrbatch import _ptr

    ldo = n if ldo is None else ldo
    _check(lib.lrb_lowrank_expand(
        ctx._h, batch, m, n, rank, _ptr(u), m * rank if su is None else su, _ptr(x),
        rank * rank if sx is None else sx, _ptr(vt), rank * n if svt is None else svt, _ptr(out),
        ldo, m * ldo if so is None else so, stream.handle if stream else None), ctx._h)
