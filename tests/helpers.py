"""Shared test helpers: host-built cases run through the C-ABI and checked
against the CPU oracle (bitwise vs its FMA chain, BASELINE's componentwise
bound vs the reference rounding)."""
from __future__ import annotations

import numpy as np

import oracle as O


def stored(order, op, rows_if_n, cols_if_n):
    """stored (rows, cols) of an operand whose op() is rows_if_n x cols_if_n"""
    return (cols_if_n, rows_if_n) if op == "T" else (rows_if_n, cols_if_n)


def min_ld(order, shape):
    r, c = shape
    return max(1, c if order == "R" else r)


def footprint(order, shape, ld):
    r, c = shape
    if r == 0 or c == 0:
        return 0
    return (r - 1) * ld + c if order == "R" else (c - 1) * ld + r


class Case:
    """A strided batch built on the host with optional ld / stride padding."""

    def __init__(self, order, opA, opB, m, n, k, batch, beta=0.0, pad=(0, 0, 0), spad=(0, 0, 0),
                 seed=0, c_fill=np.nan):
        self.order, self.opA, self.opB = order, opA, opB
        self.m, self.n, self.k, self.batch, self.beta = m, n, k, batch, beta
        rng = np.random.default_rng(seed)
        self.sa = stored(order, opA, m, k)
        self.sb = stored(order, opB, k, n)
        self.sc = (m, n)
        self.lda = min_ld(order, self.sa) + pad[0]
        self.ldb = min_ld(order, self.sb) + pad[1]
        self.ldc = min_ld(order, self.sc) + pad[2]
        self.strideA = footprint(order, self.sa, self.lda) + spad[0]
        self.strideB = footprint(order, self.sb, self.ldb) + spad[1]
        self.strideC = footprint(order, self.sc, self.ldc) + spad[2]
        nA = max(1, self.strideA * batch)
        nB = max(1, self.strideB * batch)
        nC = max(1, self.strideC * batch)
        self.A = rng.uniform(-1, 1, nA)
        self.B = rng.uniform(-1, 1, nB)
        if beta == 1.0:
            self.C0 = rng.uniform(-1, 1, nC)
        else:
            self.C0 = np.full(nC, c_fill)

    def args(self, A, B, Cm):
        return (self.order, self.opA, self.opB, self.m, self.n, self.k, self.beta, A, self.lda,
                self.strideA, B, self.ldb, self.strideB, Cm, self.ldc, self.strideC, self.batch)

    def run_device(self, ctx, variant=None, loader=None):
        dA, dB, dC = ctx.to_device(self.A), ctx.to_device(self.B), ctx.to_device(self.C0)
        ctx.set_variant_override(variant)
        ctx.set_loader(loader)
        try:
            ctx.dgemm_strided_batched(*self.args(dA, dB, dC))
            ctx.synchronize()
        finally:
            ctx.set_variant_override(None)
            ctx.set_loader(None)
        return dC.download(self.C0.size)

    def oracle(self, mode=O.FMA_CHAIN):
        out = self.C0.copy()
        O.dgemm_strided(self.order, self.opA, self.opB, self.m, self.n, self.k, self.beta, self.A,
                        self.lda, self.strideA, self.B, self.ldb, self.strideB, out, self.ldc,
                        self.strideC, self.batch, threads=4, mode=mode)
        return out

    def check(self, got, items=None):
        """bitwise vs the FMA chain (whole buffer: gaps must be untouched) and
        BASELINE's bound vs the reference rounding"""
        fma = self.oracle(O.FMA_CHAIN)
        same = np.array_equal(got, fma, equal_nan=True)
        assert same, (f"device != FMA-chain oracle: max |diff| "
                      f"{np.nanmax(np.abs(got - fma)) if got.size else 0:.3e}")
        ref = self.oracle(O.REF_COMPILED)
        worst = 0.0
        for it in (range(self.batch) if items is None else items):
            a = self.A[it * self.strideA:] if self.strideA else self.A
            b = self.B[it * self.strideB:] if self.strideB else self.B
            o = it * self.strideC
            bad, ratio = O.check_bound(self.order, self.opA, self.opB, self.m, self.n, self.k,
                                       self.beta, a, self.lda, b, self.ldb,
                                       self.C0[o:] if self.beta == 1.0 else None, got[o:],
                                       ref[o:], self.ldc)
            assert bad == 0, f"item {it}: {bad} entries outside the FP64 bound (ratio {ratio})"
            worst = max(worst, ratio)
        return worst
