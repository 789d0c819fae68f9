"""GPU: the pointer-array batch on HOST buffers (lrb_dgemm_ptr_batched_host)
against the oracle's FMA chain, bitwise. This is the reference's own calling
mode — per-item gemm_naive_raw over separately allocated host blocks
(reference blr.hpp:141-175, bench.hpp:55-77) — moved through the device in
pipelined chunks with coalesced copies."""
import zlib

import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _stored(order, op, r, c):
    return (c, r) if op == "T" else (r, c)


def _ld(order, shape, pad):
    r, c = shape
    return max(1, c if order == "R" else r) + pad


def _size(order, shape, ld):
    r, c = shape
    if r == 0 or c == 0:
        return 0
    return (r - 1) * ld + c if order == "R" else (c - 1) * ld + r


def _case(rng, order, opA, opB, dims, pad, beta):
    A, B, Cs, lda, ldb, ldc, C0 = [], [], [], [], [], [], []
    for (m, n, k) in dims:
        sa, sb, sc = _stored(order, opA, m, k), _stored(order, opB, k, n), (m, n)
        la, lb, lc = _ld(order, sa, pad), _ld(order, sb, pad), _ld(order, sc, pad)
        A.append(rng.uniform(-1, 1, max(1, _size(order, sa, la))))
        B.append(rng.uniform(-1, 1, max(1, _size(order, sb, lb))))
        c = rng.uniform(-1, 1, max(1, _size(order, sc, lc)))
        if beta == 0.0:
            c[:] = np.nan  # beta = 0 never reads C; the gaps must stay NaN
        C0.append(c.copy())
        Cs.append(c)
        lda.append(la)
        ldb.append(lb)
        ldc.append(lc)
    return A, B, Cs, lda, ldb, ldc, C0


@pytest.mark.parametrize("order", ["C", "R"])
@pytest.mark.parametrize("ops", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("beta", [0.0, 1.0])
@pytest.mark.parametrize("pad", [0, 3])
def test_ragged_pageable_blocks(ctx, order, ops, beta, pad):
    rng = np.random.default_rng(zlib.crc32(repr((order, ops, beta, pad)).encode()))
    dims = [(70, 9, 50), (130, 40, 17), (33, 64, 96), (256, 16, 256), (1, 1, 1), (0, 5, 3),
            (12, 7, 0), (65, 57, 129)]
    ms, ns, ks = [d[0] for d in dims], [d[1] for d in dims], [d[2] for d in dims]
    A, B, Cs, lda, ldb, ldc, C0 = _case(rng, order, ops[0], ops[1], dims, pad, beta)
    expect = [c.copy() for c in C0]  # the oracle writes m x n entries, gaps keep NaN
    O.dgemm_ptr(order, ops[0], ops[1], ms, ns, ks, A, lda, B, ldb, expect, ldc, beta)
    ctx.dgemm_ptr_batched_host(order, ops[0], ops[1], ms, ns, ks, A, lda, B, ldb, Cs, ldc, beta)
    for i in range(len(dims)):
        assert np.array_equal(Cs[i], expect[i], equal_nan=True), f"item {i} {dims[i]}"


def _arena_case(ctx, w, items, pinned):
    offs, (na, nb, nc) = W.variable_layout(w, items)
    if pinned:
        hA, hB, hC = ctx.pinned(na // 8), ctx.pinned(nb // 8), ctx.pinned(nc // 8)
        a, b, c = hA.array, hB.array, hC.array
        keep = (hA, hB, hC)
    else:
        a, b, c = np.empty(na // 8), np.empty(nb // 8), np.empty(nc // 8)
        keep = ()
    bs = [w.bs[i] for i in items]
    rs = [w.rs[i] for i in items]
    views_a, views_b, views_c = [], [], []
    for j, i in enumerate(items):
        bb, rr = bs[j], rs[j]
        va = a[offs[j][0] // 8: offs[j][0] // 8 + bb * bb]
        vb = b[offs[j][1] // 8: offs[j][1] // 8 + bb * rr]
        vc = c[offs[j][2] // 8: offs[j][2] // 8 + bb * rr]
        va[:] = O.fill_uniform(bb, bb, bb, 0, 1, w.seed, W.ROLE_A, i)
        vb[:] = O.fill_uniform(bb, rr, bb, 0, 1, w.seed, W.ROLE_B, i)
        vc[:] = np.nan
        views_a.append(va)
        views_b.append(vb)
        views_c.append(vc)
    return bs, rs, views_a, views_b, views_c, keep


@pytest.mark.parametrize("pinned", [True, False])
def test_cfg4_arena_prefix_bitwise(ctx, pinned):
    """a cfg4 prefix in the BASELINE layout (packed arenas, 256-B aligned
    item bases): several chunks of coalesced copies, every item bitwise the
    FMA chain"""
    w = W.get("cfg4")
    items = list(range(64))  # ~170 MB: more than one 64 MiB chunk
    bs, rs, va, vb, vc, keep = _arena_case(ctx, w, items, pinned)
    ctx.dgemm_ptr_batched_host("C", "N", "N", bs, rs, bs, va, bs, vb, bs, vc, bs, 0.0)
    expect = [np.zeros(b * r) for b, r in zip(bs, rs)]
    O.dgemm_ptr("C", "N", "N", bs, rs, bs, va, bs, vb, bs, expect, bs, 0.0, threads=8)
    for j in range(len(items)):
        assert np.array_equal(vc[j], expect[j]), f"item {items[j]}"


def test_empty_batch_is_a_noop(ctx):
    ctx.dgemm_ptr_batched_host("C", "N", "N", [], [], [], [], [], [], [], [], [], 0.0)


def test_shape_error_names_the_item(ctx):
    from paper_2311_07602_b200 import ShapeError

    a, b, c = np.zeros(16), np.zeros(16), np.zeros(16)
    with pytest.raises(ShapeError, match="item 1"):
        ctx.dgemm_ptr_batched_host("C", "N", "N", [4, 4], [4, 4], [4, 4], [a, a], [4, 2],
                                   [b, b], [4, 4], [c, c], [4, 4], 0.0)
