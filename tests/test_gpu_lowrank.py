"""GPU parity of the paper's batched low-rank product G = A_X (A_Vt B_U) B_X.

Mirrors the reference's kernel tests (proj/tests/test_kernels.cpp):
trivial all-ones (:23-28), packed == fused == reference over a rank x block
grid (:175-191), rank 32 (:193-198), determinism (:200-210), poison /
store-once (:43-48, 237-266), stale overwrite (:268-277), rank mismatch
(:279-284). Bar: bitwise equal to the oracle's three FMA-chain products; the
reference's own compare_to_reference < 1e-12 (its acceptance tolerance,
tests/acceptance.cpp:97-141) and a componentwise chained-product bound
against the reference binary's naive_multiply_batch.
"""
import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import ShapeError
from paper_2311_07602_b200 import lowrank as L

pytestmark = pytest.mark.gpu


def _check(b: L.LowRankBatch, got=None):
    got = b.g_xy_batch if got is None else got
    n, k, r = b.batch_size, b.block_size, b.rank_a
    args = (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
    fma = O.lowrank(n, k, r, *args, threads=8)
    assert np.array_equal(got, fma), f"!= FMA-chain oracle (max {np.abs(got - fma).max():.3e})"
    ref = (O.ref_lowrank(0, n, k, r, *args, workers=8) if O.ref_available()
           else O.lowrank(n, k, r, *args, threads=8, mode=O.REF_COMPILED))
    bad, ratio = O.lowrank_bound_check(n, k, r, *args, got, ref)
    assert bad == 0, f"outside the chained-product bound (ratio {ratio})"
    if O.ref_available():
        err, wi, we = O.ref_compare_to_reference(n, k, r, *args, got)
        assert err < 1e-12, f"compare_to_reference {err} at item {wi} entry {we}"


def test_trivial_all_ones(ctx):
    b = L.LowRankBatch(1, 1, 1, 1)
    b.a_vt_batch[:] = b.b_u_batch[:] = b.a_x_batch[:] = b.b_x_batch[:] = 1.0
    L.fused_multiply(b, ctx=ctx)
    assert b.g_xy_batch[0] == 1.0
    b4 = L.LowRankBatch(1, 4, 1, 1)
    for arr in (b4.a_vt_batch, b4.b_u_batch, b4.a_x_batch, b4.b_x_batch):
        arr[:] = 1.0
    L.packed_multiply(b4, ctx=ctx)
    assert b4.g_xy_batch[0] == 4.0


@pytest.mark.parametrize("rank", [1, 3, 4, 6, 8, 12, 16, 24, 32])
@pytest.mark.parametrize("block", [1, 17, 64, 256])
def test_grid_matches_reference(ctx, rank, block):
    # odd blocks take the per-item kernel, the rest the TMA+DMMA path (odd ranks
    # with B_U mapped as row pairs)
    b = L.LowRankBatch.random(7, block, rank, 1000 + rank * 10 + block)
    L.fused_multiply(b, ctx=ctx)
    _check(b)


@pytest.mark.parametrize("rank,block,batch", [(1, 64, 9), (3, 512, 41), (5, 256, 17), (7, 1024, 10),
                                              (9, 128, 33), (11, 66, 6), (15, 512, 13),
                                              (17, 256, 5), (23, 130, 7), (31, 1024, 6),
                                              (31, 34, 3), (13, 2, 4)])
def test_odd_ranks_on_the_fast_path(ctx, rank, block, batch):
    # B_U's rows are r doubles (not a 16-byte multiple): the map views each item
    # as b/2 rows of 2r, the kernel masks the columns past r. One launch,
    # bitwise the FMA-chain oracle, batches that do not fill the last CTA
    b = L.LowRankBatch.random(batch, block, rank, 77 * rank + block + batch)
    n0 = ctx.launch_count
    L.fused_multiply(b, ctx=ctx)
    assert ctx.launch_count - n0 == 1
    _check(b)


@pytest.mark.parametrize("rank,block,batch", [(8, 512, 100), (16, 1024, 33), (32, 512, 21),
                                              (32, 2048, 9), (8, 2048, 64), (16, 100, 1),
                                              (40, 128, 5), (64, 256, 6), (96, 64, 3),
                                              (128, 512, 2)])
def test_paper_shapes_and_large_ranks(ctx, rank, block, batch):
    # rank > 32 goes through three batched GEMMs
    b = L.LowRankBatch.random(batch, block, rank, rank + block + batch)
    L.packed_multiply(b, ctx=ctx)
    _check(b)


def test_device_path_and_determinism(ctx):
    b = L.LowRankBatch.random(50, 512, 16, 2222)
    d = [ctx.to_device(x) for x in (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)]
    g1, g2 = ctx.empty(b.g_xy_batch.size), ctx.empty(b.g_xy_batch.size)
    n0 = ctx.launch_count
    L.lowrank_multiply_device(ctx, 50, 512, 16, *d, g1)
    L.lowrank_multiply_device(ctx, 50, 512, 16, *d, g2)
    ctx.synchronize()
    assert ctx.launch_count - n0 == 2
    r1, r2 = g1.download(), g2.download()
    assert np.array_equal(r1, r2)
    _check(b, r1)


@pytest.mark.parametrize("eager_first", [False, True])
def test_three_gemm_path_in_a_graph(eager_first):
    # r > 32 inside stream capture: before the context workspace is sized the
    # graph owns its scratch; afterwards it references the workspace
    from paper_2311_07602_b200 import Context

    c = Context(0)
    try:
        n, blk, r = 5, 256, 48  # (ranks 64 / 96 / 128 run fused: test_gpu_lowrank_big.py)
        b = L.LowRankBatch.random(n, blk, r, 4242)
        d = [c.to_device(x) for x in (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)]
        g_eager, g_graph = c.empty(n * r * r), c.empty(n * r * r)
        s = c.stream()
        if eager_first:
            L.lowrank_multiply_device(c, n, blk, r, *d, g_eager, stream=s)
        with c.capture(s) as cap:
            L.lowrank_multiply_device(c, n, blk, r, *d, g_graph, stream=s)
        assert cap.graph.launches == 3
        for _ in range(3):
            cap.graph.launch(s)
        s.synchronize()
        got = g_graph.download()
        _check(b, got)
        if eager_first:
            assert np.array_equal(got, g_eager.download())
    finally:
        c.close()


def test_poisoned_results_are_overwritten(ctx):
    # test_kernels.cpp:43-48 / 268-277: every entry written, stale values ignored
    b = L.LowRankBatch.random(4, 32, 8, 11)
    b.g_xy_batch[:] = 1e300
    L.fused_multiply(b, ctx=ctx)
    assert np.all(np.abs(b.g_xy_batch) < 1e6)
    once = b.g_xy_batch.copy()
    L.packed_multiply(b, ctx=ctx)
    assert np.array_equal(b.g_xy_batch, once)


def test_store_once_stats(ctx):
    b = L.LowRankBatch.random(13, 256, 8, 31)
    stats = {}
    L.packed_multiply(b, stats=stats, ctx=ctx)
    assert stats["g_entry_stores"] == 13 * 8 * 8
    _check(b)


def test_rank_mismatch_rejected():
    b = L.LowRankBatch(2, 16, 4, 8)
    with pytest.raises(ShapeError, match="rank_a must equal rank_b"):
        L.fused_multiply(b)
    with pytest.raises(ShapeError, match="packed_multiply"):
        L.packed_multiply(b)


def test_negative_control():
    # tests/test_kernels.cpp:286-294: a corrupted entry is detected
    b = L.LowRankBatch.random(6, 32, 4, 13)
    args = (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
    g = O.lowrank(6, 32, 4, *args)
    g[3 * 16 + 5] += 1.0
    ref = O.lowrank(6, 32, 4, *args, mode=O.REF_COMPILED)
    bad, _ = O.lowrank_bound_check(6, 32, 4, *args, g, ref)
    assert bad == 1
    if O.ref_available():
        err, wi, we = O.ref_compare_to_reference(6, 32, 4, *args, g)
        assert err > 1e-12 and wi == 3 and we == 5


def test_graph_survives_context_workspace_growth():
    # the r > 32 path captured while the context workspace fits;
    # an eager product that needs more grows it (the old buffer is retired,
    # not freed): the graph's replays stay correct
    from paper_2311_07602_b200 import Context

    c = Context(0)
    try:
        blk, r = 256, 48
        small = L.LowRankBatch.random(3, blk, r, 5151)
        big = L.LowRankBatch.random(40, blk, r, 5152)
        ds = [c.to_device(x) for x in (small.a_vt_batch, small.b_u_batch, small.a_x_batch,
                                       small.b_x_batch)]
        db = [c.to_device(x) for x in (big.a_vt_batch, big.b_u_batch, big.a_x_batch,
                                       big.b_x_batch)]
        gs, gg, gb = c.empty(3 * r * r), c.empty(3 * r * r), c.empty(40 * r * r)
        s = c.stream()
        L.lowrank_multiply_device(c, 3, blk, r, *ds, gs, stream=s)
        with c.capture(s) as cap:
            L.lowrank_multiply_device(c, 3, blk, r, *ds, gg, stream=s)
        L.lowrank_multiply_device(c, 40, blk, r, *db, gb, stream=s)  # grows the workspace
        for _ in range(3):
            cap.graph.launch(s)
        s.synchronize()
        assert np.array_equal(gg.download(), gs.download())
        _check(big, gb.download())
    finally:
        c.close()
