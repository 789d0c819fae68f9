"""GPU parity of the batched FP64 GEMM against the CPU oracle, through the C-ABI.

Bar: bitwise equal to the oracle's FMA chain (the kernels' DMMA/DFMA rounding
is an in-order FMA chain), and inside BASELINE.json's componentwise bound
|C - C_ref| <= 4 k 2^-52 (|A||B|) against the reference binary's rounding.
Mirrors the reference's tests: known answers (tests/test_core.cpp:24-57),
packed == reference over shape grids (tests/test_kernels.cpp:175-198),
determinism (:200-210), stale-result overwrite (:268-277), negative control
(:286-294).
"""
import numpy as np
import pytest

import oracle as O
from helpers import Case
from paper_2311_07602_b200 import (DenseBlock, ShapeError, UnsupportedError, dense_gemm_naive,
                                   gemm_naive_raw, variant_names)

pytestmark = pytest.mark.gpu

OPS = [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")]


# ------------------------------------------------------------ known answers
def test_known_answers_gemm_naive_raw(ctx):
    # reference tests/test_core.cpp:24-39 through the drop-in entry point
    ident = DenseBlock.identity(3)
    m = DenseBlock(3, 3, [1, 2, 3, 4, 5, 6, 7, 8, 9])
    assert np.array_equal(dense_gemm_naive(ident, m, ctx=ctx).data, m.data)
    z = DenseBlock(2, 5)
    anyb = DenseBlock(5, 4, [3.25] * 20)
    assert np.all(dense_gemm_naive(z, anyb, ctx=ctx).data == 0.0)
    a = DenseBlock(2, 2, [1, 2, 3, 4])
    b = DenseBlock(2, 2, [5, 6, 7, 8])
    assert dense_gemm_naive(a, b, ctx=ctx).data.tolist() == [19, 22, 43, 50]


def test_known_answers_accumulate(ctx):
    # reference tests/test_core.cpp:41-49
    a = DenseBlock(2, 2, [1, 0, 0, 1])
    b = DenseBlock(2, 2, [1, 2, 3, 4])
    out = DenseBlock(2, 2, [10, 10, 10, 10])
    dense_gemm_naive(a, b, out, True, ctx=ctx)
    assert out.data.tolist() == [11, 12, 13, 14]
    dense_gemm_naive(a, b, out, False, ctx=ctx)
    assert out.data.tolist() == b.data.tolist()


def test_gemm_naive_raw_flops_counter(ctx):
    # the reference counts 2 per multiply-add inside the loop (dense.hpp:148)
    rng = np.random.default_rng(3)
    a, b = rng.uniform(-1, 1, 7 * 9), rng.uniform(-1, 1, 9 * 5)
    c = np.zeros(35)
    fl = np.array([5], dtype=np.uint64)
    gemm_naive_raw(a, b, c, 7, 9, 5, False, fl, ctx=ctx)
    assert int(fl[0]) == 5 + 2 * 7 * 9 * 5
    want = np.zeros(35)
    O.gemm_naive_raw(a, b, want, 7, 9, 5, False)  # reference rounding
    fma = np.zeros(35)
    O.dgemm_strided("R", "N", "N", 7, 5, 9, 0.0, a, 9, 0, b, 5, 0, fma, 5, 0, 1)
    assert np.array_equal(c, fma)
    bad, _ = O.check_bound("R", "N", "N", 7, 5, 9, 0.0, a, 9, b, 5, None, c, want, 5)
    assert bad == 0


def test_shape_error_text(ctx):
    # reference tests/test_core.cpp:51-57: names both shapes
    with pytest.raises(ShapeError) as e:
        dense_gemm_naive(DenseBlock(2, 3), DenseBlock(4, 2), ctx=ctx)
    assert "2x3" in str(e.value) and "4x2" in str(e.value)


def test_beta_must_be_flag(ctx):
    c = Case("C", "N", "N", 8, 8, 8, 1)
    with pytest.raises(UnsupportedError):
        ctx.dgemm_strided_batched("C", "N", "N", 8, 8, 8, 0.5, ctx.to_device(c.A), 8, 64,
                                  ctx.to_device(c.B), 8, 64, ctx.empty(64), 8, 64, 1)


# ------------------------------------------------------- variants x layouts
@pytest.mark.parametrize("loader", ["tma", "segment"])
@pytest.mark.parametrize("variant", variant_names())
@pytest.mark.parametrize("ops", OPS)
def test_every_variant_every_op_colmajor(ctx, variant, ops, loader):
    # ragged m and n, k with a tail (k % 4 == 1) across several k chunks;
    # both operand loaders (TMA tensor maps / per-segment bulk copies)
    c = Case("C", ops[0], ops[1], 138, 23, 45, 3, seed=11)
    c.check(c.run_device(ctx, variant, loader))


@pytest.mark.parametrize("variant", variant_names())
def test_every_variant_multi_tile_items(ctx, variant):
    # several row and column tiles per item, ragged in both, multiple items
    c = Case("C", "N", "N", 300, 150, 70, 3, seed=31)
    c.check(c.run_device(ctx, variant))


@pytest.mark.parametrize("variant", ["n16", "sq", "m16"])
@pytest.mark.parametrize("ops", OPS)
def test_row_major(ctx, variant, ops):
    c = Case("R", ops[0], ops[1], 29, 70, 33, 2, seed=12)
    c.check(c.run_device(ctx, variant))


@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 7, 1), (3, 1, 5), (17, 5, 13), (64, 64, 64),
                                   (128, 16, 256), (129, 17, 257), (300, 3, 2), (5, 300, 7),
                                   (8, 8, 4), (33, 65, 31)])
def test_auto_selector_shapes(ctx, shape):
    m, n, k = shape
    for order in ("C", "R"):
        c = Case(order, "N", "N", m, n, k, 4, seed=m * 1000 + n * 10 + k)
        c.check(c.run_device(ctx))


@pytest.mark.parametrize("ops", OPS)
def test_beta_one_accumulates(ctx, ops):
    c = Case("C", ops[0], ops[1], 70, 40, 37, 3, beta=1.0, seed=13)
    c.check(c.run_device(ctx))


def test_beta_zero_never_reads_c(ctx):
    # stale NaN results must be overwritten (reference tests/test_kernels.cpp:268-277)
    c = Case("C", "N", "N", 96, 16, 64, 5, c_fill=np.nan, seed=14)
    got = c.run_device(ctx)
    assert not np.isnan(got).any()
    c.check(got)


@pytest.mark.parametrize("pad", [(1, 0, 0), (0, 1, 0), (0, 0, 1), (3, 5, 7), (1, 1, 1),
                                 (2, 2, 2), (4, 6, 0)])
def test_padded_and_odd_leading_dims(ctx, pad):
    # odd ld -> misaligned column segments take the per-lane copy path;
    # even padding keeps the TMA path; gaps between columns / items must stay
    # untouched (checked bitwise)
    for ops in OPS:
        for spad in ((3, 1, 5), (2, 4, 6)):
            c = Case("C", ops[0], ops[1], 41, 19, 23, 3, pad=pad, spad=spad, seed=15)
            c.check(c.run_device(ctx))


def test_broadcast_operand_stride_zero(ctx):
    # strideA = 0: one dense block times many bases
    c = Case("C", "N", "N", 64, 16, 64, 6, seed=16)
    c.strideA = 0
    c.check(c.run_device(ctx))


def test_k_zero(ctx):
    c = Case("C", "N", "N", 33, 9, 0, 3, seed=17)
    got = c.run_device(ctx)
    assert np.all(got[np.isfinite(got)] == 0.0)
    c.check(got)
    c1 = Case("C", "N", "N", 33, 9, 0, 3, beta=1.0, seed=17)
    got1 = c1.run_device(ctx)
    assert np.array_equal(got1, c1.C0)


def test_empty_batches_are_noops(ctx):
    buf = ctx.empty(16)
    ctx.dgemm_strided_batched("C", "N", "N", 4, 4, 4, 0.0, buf, 4, 16, buf, 4, 16, buf, 4, 16, 0)
    ctx.dgemm_strided_batched("C", "N", "N", 0, 4, 4, 0.0, buf, 1, 16, buf, 4, 16, buf, 1, 16, 2)
    ctx.dgemm_strided_batched("C", "N", "N", 4, 0, 4, 0.0, buf, 4, 16, buf, 4, 16, buf, 4, 16, 2)
    ctx.synchronize()


def test_determinism_and_launch_count(ctx):
    c = Case("C", "N", "T", 128, 128, 32, 8, seed=18)
    n0 = ctx.launch_count
    g1 = c.run_device(ctx)
    g2 = c.run_device(ctx)
    assert ctx.launch_count - n0 == 2
    assert np.array_equal(g1, g2)


def test_negative_control_detects_corruption():
    # reference tests/test_kernels.cpp:286-294: the checker must flag a corrupted entry
    c = Case("C", "N", "N", 12, 6, 10, 2, seed=19)
    good = c.oracle(O.FMA_CHAIN)
    bad = good.copy()
    bad[c.strideC + 5] += 1e-9
    ref = c.oracle(O.REF_COMPILED)
    nbad, ratio = O.check_bound("C", "N", "N", 12, 6, 10, 0.0, c.A[c.strideA:], c.lda,
                                c.B[c.strideB:], c.ldb, None, bad[c.strideC:], ref[c.strideC:],
                                c.ldc)
    assert nbad == 1 and ratio > 1.0


def test_graph_capture_replays_bitwise(ctx):
    # lrb_graph_*: captured launches replay with identical results, and the
    # launch counter moves only on replay
    c = Case("C", "N", "T", 96, 80, 40, 4, seed=41)
    dA, dB, dC = ctx.to_device(c.A), ctx.to_device(c.B), ctx.to_device(c.C0)
    s = ctx.stream()
    ctx.dgemm_strided_batched(*c.args(dA, dB, dC), stream=s)  # warm (attributes)
    s.synchronize()
    dC.fill_bytes(0)
    n0 = ctx.launch_count
    with ctx.capture(s) as cap:
        ctx.dgemm_strided_batched(*c.args(dA, dB, dC), stream=s)
        ctx.dgemm_strided_batched(*c.args(dA, dB, dC), stream=s)
    g = cap.graph
    assert g.launches == 2 and ctx.launch_count == n0
    g.launch(s)
    s.synchronize()
    assert ctx.launch_count == n0 + 2
    c.check(dC.download(c.C0.size))


def test_graph_capture_of_pointer_plan(ctx):
    rng = np.random.default_rng(42)
    ms, ns, ks = [70, 130, 33], [9, 40, 64], [50, 17, 96]
    hA = [rng.uniform(-1, 1, m * k) for m, k in zip(ms, ks)]
    hB = [rng.uniform(-1, 1, k * n) for k, n in zip(ks, ns)]
    dA = [ctx.to_device(x) for x in hA]
    dB = [ctx.to_device(x) for x in hB]
    dC = [ctx.empty(m * n) for m, n in zip(ms, ns)]
    plan = ctx.ptr_plan("C", "N", "N", ms, ns, ks, dA, ms, dB, ks, dC, ms, 0.0)
    s = ctx.stream()
    plan.execute(s)
    s.synchronize()
    with ctx.capture(s) as cap:
        plan.execute(s)
    cap.graph.launch(s)
    s.synchronize()
    expect = [np.zeros(m * n) for m, n in zip(ms, ns)]
    O.dgemm_ptr("C", "N", "N", ms, ns, ks, hA, ms, hB, ks, expect, ms, 0.0)
    for i in range(3):
        assert np.array_equal(dC[i].download(ms[i] * ns[i]), expect[i])


@pytest.mark.parametrize("variant", ["q64", "n32", "n64", "m32", "s96", "n16t", None])
@pytest.mark.parametrize("k", [4, 8, 13, 16])
def test_tma_store_epilogue_short_k(ctx, variant, k):
    # beta = 0 with k <= 16 stores C through the TMA engine from shared memory
    # (variants whose C tile fits a stage): ragged tiles, even/odd m (odd m
    # keeps the register epilogue), padded ld and item gaps that must stay
    # NaN, every op combination, row-major too
    for m, n in ((70, 45), (130, 96), (41, 19)):
        for ops in OPS:
            for pad, spad in (((0, 0, 0), (0, 0, 0)), ((2, 4, 6), (2, 2, 4))):
                c = Case("C", ops[0], ops[1], m, n, k, 3, pad=pad, spad=spad, seed=m + k)
                c.check(c.run_device(ctx, variant=variant))
    r = Case("R", "N", "N", 64, 48, k, 2, seed=k)
    r.check(r.run_device(ctx, variant=variant))
