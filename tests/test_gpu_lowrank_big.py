"""GPU parity of the fused rank-64/96/128 low-rank product (csrc/lrb_lowrank_big.cu).

The paper's product G = A_X (A_Vt B_U) B_X at ranks 64, 96 and 128 runs as one launch
with T and E on chip (reference drivers fused_multiply / packed_multiply,
kernels.hpp:131-349; oracle low_rank_multiply_reference_raw,
low_rank.hpp:73-87). Bar: bitwise equal to the oracle's three FMA-chain
products and to the three-GEMM path it replaces, within the chained-product
bound of the reference binary, one launch per call, graph-capturable.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import lowrank as L

from test_gpu_lowrank import _check

pytestmark = pytest.mark.gpu

R = 128
RANKS = [64, 96, 128]


def _device(ctx, b):
    return [ctx.to_device(x) for x in (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)]


def _three_gemm(ctx, b, d, R=R):
    g = ctx.empty(b.batch_size * R * R)
    os.environ["LRB_LOWRANK_FUSED_BIG"] = "0"
    try:
        n0 = ctx.launch_count
        L.lowrank_multiply_device(ctx, b.batch_size, b.block_size, R, *d, g)
        assert ctx.launch_count - n0 == 3
        ctx.synchronize()
    finally:
        del os.environ["LRB_LOWRANK_FUSED_BIG"]
    return g.download()


# batch below / above the grid (148 CTAs: several items per CTA, the ring
# running across item boundaries; 296 at rank 64), the smallest eligible block
# (three phase-1 chunks: 48), the paper's blocks
@pytest.mark.parametrize("R", RANKS)
@pytest.mark.parametrize("batch,block", [(1, 48), (3, 64), (7, 1024), (2, 2048), (300, 48),
                                         (160, 112), (700, 64)])
def test_fused_matches_oracle_and_three_gemms(ctx, R, batch, block):
    b = L.LowRankBatch.random(batch, block, R, 9000 + batch + block + R)
    d = _device(ctx, b)
    g = ctx.empty(batch * R * R)
    n0 = ctx.launch_count
    L.lowrank_multiply_device(ctx, batch, block, R, *d, g)
    ctx.synchronize()
    assert ctx.launch_count - n0 == 1, f"rank {R} runs as one launch"
    got = g.download()
    _check(b, got)
    assert np.array_equal(got, _three_gemm(ctx, b, d, R))


@pytest.mark.parametrize("R", RANKS)
def test_fused_unaligned_output(ctx, R):
    # G at an 8-byte and a 16-byte offset: the scalar and 16-byte store forms
    b = L.LowRankBatch.random(4, 128, R, 9100 + R)
    d = _device(ctx, b)
    n = 4 * R * R
    for off in (1, 2):
        buf = ctx.empty(n + 4)
        buf.fill_bytes(0)
        n0 = ctx.launch_count
        L.lowrank_multiply_device(ctx, 4, 128, R, *d, buf.ptr + 8 * off)
        assert ctx.launch_count - n0 == 1
        ctx.synchronize()
        all_ = buf.download()
        assert not all_[:off].any() and not all_[off + n:].any(), "wrote outside G"
        _check(b, all_[off:off + n].copy())


@pytest.mark.parametrize("R", RANKS)
def test_fused_in_a_graph_and_repeatable(R):
    from paper_2311_07602_b200 import Context

    c = Context(0)
    try:
        b = L.LowRankBatch.random(350, 64, R, 9200 + R)
        d = _device(c, b)
        g_eager, g_graph = c.empty(350 * R * R), c.empty(350 * R * R)
        s = c.stream()
        L.lowrank_multiply_device(c, 350, 64, R, *d, g_eager, stream=s)
        with c.capture(s) as cap:
            L.lowrank_multiply_device(c, 350, 64, R, *d, g_graph, stream=s)
        assert cap.graph.launches == 1
        for _ in range(3):
            cap.graph.launch(s)
        s.synchronize()
        got = g_graph.download()
        assert np.array_equal(got, g_eager.download())
        _check(b, got)
    finally:
        c.close()


@pytest.mark.parametrize("R,block", [(128, 40), (96, 40), (64, 40), (64, 32)])
def test_ineligible_blocks_keep_three_gemms(ctx, R, block):
    # a block that is not a multiple of the phase-1 chunk (16) or shorter than
    # three chunks takes the three-GEMM path (3 launches)
    b = L.LowRankBatch.random(2, block, R, 9300 + R)
    d = _device(ctx, b)
    g = ctx.empty(2 * R * R)
    n0 = ctx.launch_count
    L.lowrank_multiply_device(ctx, 2, block, R, *d, g)
    ctx.synchronize()
    assert ctx.launch_count - n0 == 3
    _check(b, g.download())
