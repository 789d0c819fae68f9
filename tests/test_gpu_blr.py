"""GPU BLR multi-RHS matvec (reference blr.hpp:141-202; tests/test_blr.cpp).

Bitwise equal to the FMA-chain restatement of blr_matvec_naive; against the
reference binary's blr_matvec (packed path) and its dense reconstruction
within the reference's own tolerance (max_rel < 1e-10, test_blr.cpp:12-22)."""
import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import DenseBlock, ShapeError
from paper_2311_07602_b200 import blr as B
from paper_2311_07602_b200 import lowrank as L

pytestmark = pytest.mark.gpu


def max_rel(got, expect):
    # tests/test_blr.cpp:12-22
    rms = np.sqrt(np.mean(expect * expect))
    floor = rms if rms > 0 else 1.0
    return float(np.max(np.abs(got - expect) / np.maximum(np.abs(expect), floor)))


def _rhs(n, nrhs, seed):
    return DenseBlock(n, nrhs, L._uniform_vec(seed * 7919 + 1, 0, np.arange(n * nrhs, dtype=np.uint64)))


def _check(m, rhs, y):
    diag, u, x, vt = m.packed_arrays()
    args = (m.n, m.block_size, m.rank, diag, u, x, vt, rhs.data, rhs.cols)
    fma = O.blr_matvec(*args)
    assert np.array_equal(y.data, fma), f"!= FMA-chain oracle ({np.abs(y.data - fma).max():.3e})"
    if O.ref_available():
        assert max_rel(y.data, O.ref_blr_matvec(1, *args)) < 1e-11  # blr_matvec_naive
        assert max_rel(y.data, O.ref_blr_matvec(0, *args)) < 1e-10  # packed blr_matvec
        assert max_rel(y.data, O.ref_blr_matvec(2, *args)) < 1e-10  # dense reconstruction
    else:
        assert max_rel(y.data, O.blr_matvec(*args, mode=O.REF_COMPILED)) < 1e-11


def test_identity_like_maps_rhs_to_itself(ctx):
    # test_blr.cpp "identity-like BLR maps rhs to itself"
    block, tiles, rank = 16, 3, 4
    m = B.BlrMatrix.random(block * tiles, block, rank, 5)
    for t in range(tiles):
        m.diagonal[t] = DenseBlock.identity(block)
    for tile in m.off_diagonal:
        tile.u[:] = 0.0
        tile.x[:] = 0.0
        tile.vt[:] = 0.0
    rhs = _rhs(block * tiles, 2, 7)
    y = B.blr_matvec(m, rhs, ctx=ctx)
    assert np.array_equal(y.data, rhs.data)


@pytest.mark.parametrize("tiles,rank,nrhs,block", [(2, 4, 8, 32), (4, 4, 1, 24), (4, 8, 8, 24),
                                                   (16, 4, 1, 24), (16, 8, 8, 24), (5, 4, 6, 20),
                                                   (3, 8, 11, 16), (1, 4, 3, 16), (8, 16, 16, 64),
                                                   # r^2 + r nrhs > 512: the register-blocked
                                                   # coupling kernel instead of warp-per-item
                                                   (3, 24, 8, 48), (2, 16, 24, 32),
                                                   # b a multiple of 64, even nrhs <= 16: the
                                                   # row step reads rhs itself (BlrRowProblem)
                                                   (4, 8, 8, 64), (3, 16, 2, 128), (5, 8, 4, 64),
                                                   (6, 16, 16, 128)])
def test_grids_match_reference(ctx, tiles, rank, nrhs, block):
    m = B.BlrMatrix.random(tiles * block, block, rank, 100 + tiles + rank + nrhs)
    rhs = _rhs(tiles * block, nrhs, 17 + nrhs)
    _check(m, rhs, B.blr_matvec(m, rhs, ctx=ctx))


def test_linearity_and_reuse(ctx):
    # test_blr.cpp "linearity in the right-hand side" (+ nrhs changes reuse the upload)
    block, tiles, rank, nrhs = 24, 4, 8, 3
    m = B.BlrMatrix.random(tiles * block, block, rank, 23)
    r1, r2 = _rhs(tiles * block, nrhs, 29), _rhs(tiles * block, nrhs, 30)
    a, b = 1.75, -0.5
    mix = DenseBlock(tiles * block, nrhs, a * r1.data + b * r2.data)
    y_mix = B.blr_matvec(m, mix, ctx=ctx)
    y1, y2 = B.blr_matvec(m, r1, ctx=ctx), B.blr_matvec(m, r2, ctx=ctx)
    assert max_rel(y_mix.data, a * y1.data + b * y2.data) < 1e-10
    _check(m, r1, y1)
    r5 = _rhs(tiles * block, 5, 31)
    _check(m, r5, B.blr_matvec(m, r5, ctx=ctx))


def test_paper_scale_rank8_8rhs(ctx):
    # the paper's BLR experiment shape (rank 8, 8 RHS), n = 8192, block 512
    m = B.BlrMatrix.random(8192, 512, 8, 3)
    rhs = _rhs(8192, 8, 4)
    y = B.blr_matvec(m, rhs, ctx=ctx)
    diag, u, x, vt = m.packed_arrays()
    fma = O.blr_matvec(8192, 512, 8, diag, u, x, vt, rhs.data, 8)
    assert np.array_equal(y.data, fma)


def test_constraints():
    with pytest.raises(ShapeError, match="not a multiple"):
        B.BlrMatrix(100, 16, 4)
    with pytest.raises(ShapeError, match="rank must be in"):
        B.BlrMatrix(64, 16, 17)
    m = B.BlrMatrix.random(64, 16, 4, 1)
    with pytest.raises(ShapeError, match="rhs has"):
        B.blr_matvec(m, DenseBlock(32, 2))


@pytest.mark.parametrize("tiles,rank,nrhs,block", [(4, 8, 8, 64), (3, 8, 6, 20)])
def test_device_matvec_in_a_graph_replayed(ctx, tiles, rank, nrhs, block):
    # the three launches under stream capture (programmatic-dependent edges,
    # the row step's deferred wait), replayed back to back: every replay
    # bitwise equal to the eager device result and the FMA-chain oracle
    from paper_2311_07602_b200.lrbatch import _check as check, lib

    m = B.BlrMatrix.random(tiles * block, block, rank, 61 + tiles)
    rhs = _rhs(tiles * block, nrhs, 5)
    h = m.device_handle(ctx)
    s = ctx.stream()
    d_rhs = ctx.to_device(rhs.data)
    y_eager, y_graph = ctx.empty(rhs.data.size), ctx.empty(rhs.data.size)
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_eager.ptr, s.handle), ctx._h)
    s.synchronize()
    with ctx.capture(s) as cap:
        check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_graph.ptr, s.handle),
              ctx._h)
    assert cap.graph.launches in (1, 3)  # the fused single launch, or the three-launch form
    want = y_eager.download(rhs.data.size)
    _check(m, rhs, DenseBlock(rhs.rows, rhs.cols, want))
    for _ in range(5):
        y_graph.fill_bytes(0)
        ctx.synchronize()
        cap.graph.launch(s)
        cap.graph.launch(s)
        s.synchronize()
        assert np.array_equal(y_graph.download(rhs.data.size), want)


def test_graph_survives_workspace_growth_and_other_streams(ctx):
    # a matvec captured with one nrhs, then eager calls with a
    # larger nrhs (the workspace grows: the old buffers are retired, not
    # freed) and on a second stream; every replay of the graph still equals
    # the eager result
    from paper_2311_07602_b200.lrbatch import _check as check, lib

    tiles, block, rank = 4, 64, 8
    m = B.BlrMatrix.random(tiles * block, block, rank, 77)
    h = m.device_handle(ctx)
    s1, s2 = ctx.stream(), ctx.stream()
    small, big = _rhs(tiles * block, 4, 1), _rhs(tiles * block, 16, 2)
    d_small, d_big = ctx.to_device(small.data), ctx.to_device(big.data)
    y_eager, y_graph = ctx.empty(small.data.size), ctx.empty(small.data.size)
    y_big1, y_big2 = ctx.empty(big.data.size), ctx.empty(big.data.size)
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_small.ptr, 4, y_eager.ptr, s1.handle), ctx._h)
    s1.synchronize()
    with ctx.capture(s1) as cap:
        check(lib.lrb_blr_matvec_device(ctx._h, h, d_small.ptr, 4, y_graph.ptr, s1.handle),
              ctx._h)
    want = y_eager.download(small.data.size)
    # grow the workspace, then alternate streams (ordered by the matrix's event)
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_big.ptr, 16, y_big1.ptr, s1.handle), ctx._h)
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_big.ptr, 16, y_big2.ptr, s2.handle), ctx._h)
    for _ in range(3):
        cap.graph.launch(s1)
    ctx.synchronize()
    assert np.array_equal(y_graph.download(small.data.size), want)
    _check(m, big, DenseBlock(big.rows, big.cols, y_big1.download(big.data.size)))
    assert np.array_equal(y_big1.download(big.data.size), y_big2.download(big.data.size))


FUSED_SHAPES = [(2, 8, 10, 64), (4, 16, 16, 64), (5, 4, 12, 128), (8, 16, 12, 64), (3, 8, 16, 128),
                (17, 8, 14, 64), (6, 16, 10, 256), (9, 4, 10, 192), (33, 16, 16, 64),
                # up to 8 right-hand sides: the m8 tile
                (4, 8, 8, 64), (5, 16, 8, 128), (3, 4, 6, 64), (9, 8, 2, 128), (17, 16, 4, 64),
                (8, 8, 8, 512),
                # rank 32: X_ij read straight from global memory by the coupling warp
                (3, 32, 16, 64), (5, 32, 8, 128), (9, 32, 10, 256), (17, 32, 2, 64)]


@pytest.mark.parametrize("tiles,rank,nrhs,block", [(4, 8, 1, 64), (9, 16, 1, 128), (5, 8, 3, 128),
                                                   (6, 32, 7, 64), (17, 16, 15, 64),
                                                   (3, 4, 5, 96)])
def test_fused_matvec_odd_rhs_counts(ctx, monkeypatch, tiles, rank, nrhs, block):
    # an odd count (the plain matvec first of all) runs the fused launch on
    # copies padded with one zero column: three launches (pad, fused, unpad),
    # results bitwise the three-launch form's and the oracle's; replayed from
    # a graph
    from paper_2311_07602_b200.lrbatch import _check as check, lib

    m = B.BlrMatrix.random(tiles * block, block, rank, 500 + tiles + rank)
    rhs = _rhs(tiles * block, nrhs, 91 + nrhs)
    h = m.device_handle(ctx)
    s = ctx.stream()
    d_rhs = ctx.to_device(rhs.data)
    y_f, y_3 = ctx.empty(rhs.data.size), ctx.empty(rhs.data.size)
    n0 = ctx.launch_count
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_f.ptr, s.handle), ctx._h)
    s.synchronize()
    assert ctx.launch_count - n0 == 3
    monkeypatch.setenv("LRB_BLR_FUSED", "0")
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_3.ptr, s.handle), ctx._h)
    s.synchronize()
    monkeypatch.delenv("LRB_BLR_FUSED")
    got = y_f.download(rhs.data.size)
    assert np.array_equal(got, y_3.download(rhs.data.size))
    _check(m, rhs, DenseBlock(rhs.rows, rhs.cols, got))
    with ctx.capture(s) as cap:
        check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_f.ptr, s.handle), ctx._h)
    for _ in range(2):
        y_f.fill_bytes(0)
        ctx.synchronize()
        cap.graph.launch(s)
        s.synchronize()
        assert np.array_equal(y_f.download(rhs.data.size), got)


@pytest.mark.parametrize("tiles,rank,nrhs,block", [(5, 8, 18, 64), (9, 16, 32, 128), (4, 32, 24, 64),
                                                   (6, 16, 33, 96), (3, 16, 64, 64), (7, 4, 47, 32),
                                                   (5, 32, 47, 64)])
def test_fused_matvec_column_ranges_beyond_16_rhs(ctx, monkeypatch, tiles, rank, nrhs, block):
    # 17..64 right-hand sides: the fused launch once per column range of 16
    # (rhs and y addressed with the full row pitch), odd counts padded first;
    # bitwise the three-launch form and the oracle
    from paper_2311_07602_b200.lrbatch import _check as check, lib

    m = B.BlrMatrix.random(tiles * block, block, rank, 700 + tiles + rank)
    rhs = _rhs(tiles * block, nrhs, 17 + nrhs)
    h = m.device_handle(ctx)
    s = ctx.stream()
    d_rhs = ctx.to_device(rhs.data)
    y_f, y_3 = ctx.empty(rhs.data.size), ctx.empty(rhs.data.size)
    n0 = ctx.launch_count
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_f.ptr, s.handle), ctx._h)
    s.synchronize()
    even = nrhs + (nrhs & 1)
    # (ranks below 16 keep the three launches there: measured faster)
    core = (even + 15) // 16 if rank >= 16 else 3
    assert ctx.launch_count - n0 == core + (2 if nrhs & 1 else 0)
    monkeypatch.setenv("LRB_BLR_FUSED", "0")
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_3.ptr, s.handle), ctx._h)
    s.synchronize()
    monkeypatch.delenv("LRB_BLR_FUSED")
    got = y_f.download(rhs.data.size)
    assert np.array_equal(got, y_3.download(rhs.data.size))
    _check(m, rhs, DenseBlock(rhs.rows, rhs.cols, got))


@pytest.mark.parametrize("tiles,rank,block", [(9, 16, 128), (6, 32, 64), (17, 8, 64)])
def test_fused_matvec_changing_rhs_counts_on_one_matrix(ctx, monkeypatch, tiles, rank, block):
    # one matrix, a sequence of calls with different right-hand-side counts
    # (the m16 and the m8 tile share the matrix's sync words: ready counts that
    # only grow, one epoch word), with three-launch calls in between (they
    # leave the words alone): every fused result bitwise the three-launch one
    from paper_2311_07602_b200.lrbatch import _check as check, lib

    m = B.BlrMatrix.random(tiles * block, block, rank, 900 + tiles)
    h = m.device_handle(ctx)
    s = ctx.stream()
    for rep, nrhs in enumerate([16, 8, 16, 2, 1, 10, 10, 3, 4, 16]):
        rhs = _rhs(tiles * block, nrhs, 70 + rep)
        d_rhs = ctx.to_device(rhs.data)
        y_f, y_3 = ctx.empty(rhs.data.size), ctx.empty(rhs.data.size)
        n0 = ctx.launch_count
        check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_f.ptr, s.handle), ctx._h)
        s.synchronize()
        assert ctx.launch_count - n0 == (3 if nrhs % 2 else 1)
        monkeypatch.setenv("LRB_BLR_FUSED", "0")
        check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_3.ptr, s.handle), ctx._h)
        s.synchronize()
        monkeypatch.delenv("LRB_BLR_FUSED")
        assert np.array_equal(y_f.download(rhs.data.size), y_3.download(rhs.data.size)), (rep, nrhs)


@pytest.mark.parametrize("tiles,rank,nrhs,block", FUSED_SHAPES)
def test_fused_matvec_equals_three_launch_form(ctx, monkeypatch, tiles, rank, nrhs, block):
    # the single persistent launch (W tiles with the coupling folded in, row
    # tiles waiting on per-row ready counts) against the three-launch form and
    # the FMA-chain oracle, bitwise; replayed from a graph (the tickets and
    # ready counts reset themselves)
    from paper_2311_07602_b200.lrbatch import _check as check, lib

    m = B.BlrMatrix.random(tiles * block, block, rank, 300 + tiles + rank)
    rhs = _rhs(tiles * block, nrhs, 41 + nrhs)
    h = m.device_handle(ctx)
    s = ctx.stream()
    d_rhs = ctx.to_device(rhs.data)
    y_f, y_3 = ctx.empty(rhs.data.size), ctx.empty(rhs.data.size)
    n0 = ctx.launch_count
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_f.ptr, s.handle), ctx._h)
    s.synchronize()
    assert ctx.launch_count - n0 == 1
    monkeypatch.setenv("LRB_BLR_FUSED", "0")
    check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_3.ptr, s.handle), ctx._h)
    s.synchronize()
    monkeypatch.delenv("LRB_BLR_FUSED")
    got = y_f.download(rhs.data.size)
    assert np.array_equal(got, y_3.download(rhs.data.size))
    _check(m, rhs, DenseBlock(rhs.rows, rhs.cols, got))
    with ctx.capture(s) as cap:
        check(lib.lrb_blr_matvec_device(ctx._h, h, d_rhs.ptr, nrhs, y_f.ptr, s.handle), ctx._h)
    assert cap.graph.launches == 1
    for _ in range(3):
        y_f.fill_bytes(0)
        ctx.synchronize()
        cap.graph.launch(s)
        cap.graph.launch(s)
        s.synchronize()
        assert np.array_equal(y_f.download(rhs.data.size), got)
