"""GPU parity of the row-panel kernel (p256, csrc/lrb_panel.cu): short-k
strided products C_i = U_i op(V_i) (+ C_i), the low-rank expansion shape of
BASELINE cfg2 (reference blr.hpp:75-78, dense.hpp:43-56 per item).

Bar as everywhere: bitwise equal to the oracle's in-order FMA chain and inside
BASELINE's componentwise bound against the reference rounding. Covers ragged
rows (partial 256-row units and half panels), ragged columns (partial 32-column
chunks), every k in 1..32 class (DMMA steps + scalar tail), beta = 1, padded
ld / strides, broadcast operands, row-major calls, long unit sequences per CTA
(ring and double-buffer wrap).
"""
import os

import numpy as np
import pytest

from helpers import Case

pytestmark = pytest.mark.gpu


def panel_case(order, opA, opB, m, n, k, batch, pad=(0, 0, 0), spad=(0, 0, 0), **kw):
    """a Case whose leading dimensions and strides are even (TMA needs
    16-byte strides; odd ones take the tile kernel's segment loader)"""
    c = Case(order, opA, opB, m, n, k, batch, pad=pad, spad=spad, **kw)
    pad = (pad[0] + c.lda % 2, pad[1] + c.ldb % 2, pad[2])
    c = Case(order, opA, opB, m, n, k, batch, pad=pad, spad=spad, **kw)
    spad = (spad[0] + c.strideA % 2, spad[1] + c.strideB % 2, spad[2])
    return Case(order, opA, opB, m, n, k, batch, pad=pad, spad=spad, **kw)


def run_panel(ctx, c, flags=None):
    old = os.environ.get("LRB_DEBUG_FLAGS")
    if flags is not None:
        os.environ["LRB_DEBUG_FLAGS"] = str(flags)
    try:
        got = c.run_device(ctx, "p256")
    finally:
        if flags is not None:
            if old is None:
                os.environ.pop("LRB_DEBUG_FLAGS", None)
            else:
                os.environ["LRB_DEBUG_FLAGS"] = old
    assert ctx.last_variant == "p256"
    return got


@pytest.mark.parametrize("opB", ["N", "T"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 7, 8, 13, 16, 29, 31, 32])
def test_panel_every_k(ctx, opB, k):
    c = panel_case("C", "N", opB, 300, 70, k, 3, seed=100 + k)
    c.check(run_panel(ctx, c))


@pytest.mark.parametrize("m,n", [(1, 1), (7, 33), (128, 32), (129, 31), (200, 96), (256, 64),
                                 (257, 65), (384, 130), (512, 512), (513, 17)])
@pytest.mark.parametrize("opB", ["N", "T"])
def test_panel_ragged_shapes(ctx, m, n, opB):
    c = panel_case("C", "N", opB, m, n, 32, 2, seed=m * 7 + n)
    c.check(run_panel(ctx, c))


@pytest.mark.parametrize("opB", ["N", "T"])
def test_panel_beta_one(ctx, opB):
    c = panel_case("C", "N", opB, 260, 50, 17, 3, beta=1.0, seed=5)
    c.check(run_panel(ctx, c))


def test_panel_padded_ld_and_strides(ctx):
    c = panel_case("C", "N", "T", 270, 45, 24, 3, pad=(2, 4, 6), spad=(10, 6, 8), seed=9)
    c.check(run_panel(ctx, c))


@pytest.mark.parametrize("opA", ["N", "T"])
def test_panel_row_major_calls(ctx, opA):
    # row-major C = op(A) op(B) runs as column-major C^T = op(B)^T op(A)^T:
    # the panel serves it when op(B) = N in the caller's terms
    c = panel_case("R", opA, "N", 40, 300, 32, 3, seed=12)
    c.check(run_panel(ctx, c))


def test_panel_long_sequences_wrap_ring_and_buffers(ctx):
    # 600 items x 2 units over <= 148 CTAs: ~8 units per CTA, 3 chunks each
    # (odd: the groups alternate parity across units)
    c = Case("C", "N", "T", 320, 90, 32, 600, seed=21)
    c.check(run_panel(ctx, c), items=range(0, 600, 37))


def test_panel_many_units_per_cta(ctx):
    # 320 units over <= 148 CTAs, 5 chunks per unit
    c = Case("C", "N", "T", 512, 160, 32, 160, seed=33)
    c.check(run_panel(ctx, c), items=range(0, 160, 13))


def test_panel_broadcast_operand(ctx):
    # strideB = 0: one V for every item
    c = Case("C", "N", "T", 256, 64, 32, 4, seed=44)
    c.strideB = 0
    c.check(run_panel(ctx, c))


def test_panel_falls_back_where_it_does_not_serve(ctx):
    # op(A) = T, or k > 32: the forced p256 falls back to the tile kernel
    c = Case("C", "T", "N", 260, 40, 20, 2, seed=2)
    c.check(c.run_device(ctx, "p256"))
    assert ctx.last_variant != "p256"
    c = Case("C", "N", "N", 260, 40, 33, 2, seed=3)
    c.check(c.run_device(ctx, "p256"))
    assert ctx.last_variant != "p256"


def test_panel_is_the_automatic_choice_for_cfg2_shape(ctx):
    c = Case("C", "N", "T", 512, 512, 32, 300, seed=1)
    got = c.run_device(ctx)
    assert ctx.last_variant == "p256"
    c.check(got, items=[0, 1, 150, 299])


@pytest.mark.parametrize("beta,m", [(1.0, 300), (0.0, 302)])
def test_panel_short_k_forced(ctx, beta, m):
    # k <= 16 is not the automatic choice (write-bound: the tile kernel's
    # TMA-store epilogue wins) but the forced panel stays exact there
    c = panel_case("C", "N", "T", m, 64, 8, 3, beta=beta, pad=(0, 0, 6), spad=(0, 0, 10), seed=7)
    c.check(run_panel(ctx, c))
