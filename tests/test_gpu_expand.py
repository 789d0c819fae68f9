"""GPU low-rank expansion (U X) Vt and BLR dense reconstruction
(reference blr.hpp:62-86; tests/test_blr.cpp's reconstruct_dense oracle use).

Bitwise equal to the FMA-chain restatement; against the reference binary's
dense_gemm_naive(dense_gemm_naive(U, X), Vt) and reconstruct_dense within the
chained-product bound 4 (2r) 2^-52 (|U||X||Vt|)."""
import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import DenseBlock
from paper_2311_07602_b200 import blr as B
from paper_2311_07602_b200 import lowrank as L

pytestmark = pytest.mark.gpu


def _operands(batch, m, n, r, seed):
    g = lambda role, size: L._uniform_vec(seed * 31 + role, 0, np.arange(size, dtype=np.uint64))  # noqa
    return g(1, batch * m * r), g(2, batch * r * r), g(3, batch * r * n)


def _bound_check(got, ref, batch, m, n, r, u, x, vt):
    mags = O.lowrank_expand(batch, m, n, r, np.abs(u), np.abs(x), np.abs(vt))
    bound = 4.0 * (2 * r) * 2.0 ** -52 * mags
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) / (bound + 1e-300)))


@pytest.mark.parametrize("batch,m,n,r", [(3, 512, 512, 32), (5, 17, 13, 5), (4, 64, 48, 8),
                                         (2, 100, 100, 1), (3, 33, 65, 33), (7, 256, 256, 16),
                                         (1, 1, 1, 1), (2, 130, 70, 64)])
def test_expand_matches_oracle_and_reference(ctx, batch, m, n, r):
    u, x, vt = _operands(batch, m, n, r, batch + m + r)
    got = B.lowrank_expand(u, x, vt, batch, m, n, r, ctx=ctx)
    assert np.array_equal(got, O.lowrank_expand(batch, m, n, r, u, x, vt)), "!= FMA-chain oracle"
    ref = (O.ref_lowrank_expand(batch, m, n, r, u, x, vt) if O.ref_available()
           else O.lowrank_expand(batch, m, n, r, u, x, vt, mode=O.REF_COMPILED))
    _bound_check(got, ref, batch, m, n, r, u, x, vt)


def test_expand_padded_output_leaves_gaps(ctx):
    batch, m, n, r, ldo = 3, 40, 24, 8, 30
    so = m * ldo + 7
    u, x, vt = _operands(batch, m, n, r, 9)
    du, dx, dvt = ctx.to_device(u), ctx.to_device(x), ctx.to_device(vt)
    size = (batch - 1) * so + (m - 1) * ldo + n
    poison = np.full(size, 12345.0)
    dout = ctx.to_device(poison)
    B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, dout, ldo=ldo, so=so)
    ctx.synchronize()
    got = dout.download()
    want = O.lowrank_expand(batch, m, n, r, u, x, vt, ldo=ldo, so=so, out=poison.copy())
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,block,rank", [(96, 32, 6), (64, 16, 4), (256, 64, 16), (48, 48, 8),
                                          (120, 24, 5), (1024, 128, 8), (256, 32, 24), (512, 64, 32)])
def test_reconstruct_dense_matches_reference(ctx, n, block, rank):
    m = B.BlrMatrix.random(n, block, rank, n + rank)
    full = m.reconstruct_dense(ctx=ctx)
    diag, u, x, vt = m.packed_arrays()
    assert np.array_equal(full.data, O.blr_reconstruct(n, block, rank, diag, u, x, vt))
    if O.ref_available():
        ref = O.ref_blr_reconstruct(n, block, rank, diag, u, x, vt)
        err = np.abs(full.data - ref)
        assert float(err.max()) <= 4 * 2 * rank * 2.0 ** -52 * 8 * rank * rank
    # the diagonal tiles are copies
    for t in range(n // block):
        tile = full.data.reshape(n, n)[t * block:(t + 1) * block, t * block:(t + 1) * block]
        assert np.array_equal(tile.ravel(), m.diagonal[t].data)


def test_reconstruct_dense_device_buffer_reuse(ctx):
    # the tile plan is cached per output buffer; a second buffer rebuilds it
    m = B.BlrMatrix.random(128, 32, 4, 5)
    a, b = ctx.empty(128 * 128), ctx.empty(128 * 128)
    m.reconstruct_dense_device(ctx, a)
    m.reconstruct_dense_device(ctx, b)
    m.reconstruct_dense_device(ctx, a)
    ctx.synchronize()
    assert np.array_equal(a.download(), b.download())


def test_reconstructed_matrix_times_rhs_is_the_matvec(ctx):
    # test_blr.cpp: blr_matvec == dense_gemm_naive(reconstruct_dense(), rhs)
    n, block, rank, nrhs = 192, 32, 6, 5
    m = B.BlrMatrix.random(n, block, rank, 77)
    rhs = DenseBlock(n, nrhs, L._uniform_vec(5, 0, np.arange(n * nrhs, dtype=np.uint64)))
    y = B.blr_matvec(m, rhs, ctx=ctx)
    full = m.reconstruct_dense(ctx=ctx).data.reshape(n, n)
    expect = full @ rhs.data.reshape(n, nrhs)
    rms = np.sqrt(np.mean(expect * expect))
    assert np.max(np.abs(y.data.reshape(n, nrhs) - expect) / np.maximum(np.abs(expect), rms)) < 1e-10


def test_expand_in_a_graph(ctx):
    batch, m, n, r = 4, 128, 96, 16
    u, x, vt = _operands(batch, m, n, r, 3)
    du, dx, dvt = ctx.to_device(u), ctx.to_device(x), ctx.to_device(vt)
    out = ctx.empty(batch * m * n)
    s = ctx.stream()
    B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, out, stream=s)  # sizes workspace
    s.synchronize()
    out2 = ctx.empty(batch * m * n)
    with ctx.capture(s) as cap:
        B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, out2, stream=s)
    assert cap.graph.launches == 2
    cap.graph.launch(s)
    s.synchronize()
    assert np.array_equal(out.download(), out2.download())


@pytest.mark.parametrize("n,block,rank", [(512, 256, 8), (768, 256, 16), (2048, 512, 16),
                                          (1024, 512, 8),
                                          # even ranks below the template rank (8 or 16)
                                          (768, 256, 12), (512, 256, 6), (1024, 256, 2),
                                          (1536, 512, 14), (768, 256, 10), (512, 256, 4)])
def test_reconstruct_dense_streaming_kernel(ctx, monkeypatch, n, block, rank):
    # shapes the write-streaming off-diagonal kernel serves (b a multiple of
    # 256, even r <= 16: a rank below 8 / 16 rides on the boxes' zero fill and
    # masked X reads): bitwise the FMA-chain oracle and the UX + tile form
    m = B.BlrMatrix.random(n, block, rank, 3 * n + rank)
    out, alt = ctx.empty(n * n), ctx.empty(n * n)
    out.fill_bytes(0xFF)
    n0 = ctx.launch_count
    m.reconstruct_dense_device(ctx, out)
    ctx.synchronize()
    assert ctx.launch_count - n0 == 2  # the diagonal copy + one streaming launch
    monkeypatch.setenv("LRB_BLR_RECON", "0")
    m.reconstruct_dense_device(ctx, alt)
    ctx.synchronize()
    got = out.download(n * n)
    assert np.array_equal(got, alt.download(n * n))
    diag, u, x, vt = m.packed_arrays()
    assert np.array_equal(got, O.blr_reconstruct(n, block, rank, diag, u, x, vt))


@pytest.mark.parametrize("batch,m,n,r,pad", [(3, 64, 256, 8, 0), (2, 128, 512, 16, 0),
                                             (5, 192, 256, 16, 6), (1, 512, 768, 8, 2),
                                             (4, 128, 256, 12, 0), (3, 64, 512, 6, 4),
                                             (2, 256, 256, 2, 0), (3, 128, 512, 14, 2),
                                             (5, 64, 256, 10, 0), (2, 192, 256, 4, 6)])
def test_expand_streaming_kernel(ctx, monkeypatch, batch, m, n, r, pad):
    # even ranks up to 16 with 64-row, 256-column items: one write-streaming launch
    # (UX on chip), bitwise the FMA-chain oracle and the two-GEMM form, padded
    # leading dimensions and item strides left untouched
    u, x, vt = _operands(batch, m, n, r, 7 * m + r)
    du, dx, dvt = ctx.to_device(u), ctx.to_device(x), ctx.to_device(vt)
    ldo = n + pad
    so = m * ldo + 2 * pad
    size = (batch - 1) * so + (m - 1) * ldo + n
    poison = np.full(size, -7.5)
    dout, dalt = ctx.to_device(poison), ctx.to_device(poison)
    n0 = ctx.launch_count
    B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, dout, ldo=ldo, so=so)
    ctx.synchronize()
    assert ctx.launch_count - n0 == 1
    monkeypatch.setenv("LRB_EXPAND_STREAM", "0")
    n0 = ctx.launch_count
    B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, dalt, ldo=ldo, so=so)
    ctx.synchronize()
    assert ctx.launch_count - n0 == 2
    got = dout.download()
    assert np.array_equal(got, dalt.download())
    want = O.lowrank_expand(batch, m, n, r, u, x, vt, ldo=ldo, so=so, out=poison.copy())
    assert np.array_equal(got, want)


def test_expand_streaming_kernel_in_a_graph(ctx):
    batch, m, n, r = 3, 128, 256, 16
    u, x, vt = _operands(batch, m, n, r, 5)
    du, dx, dvt = ctx.to_device(u), ctx.to_device(x), ctx.to_device(vt)
    out, out2 = ctx.empty(batch * m * n), ctx.empty(batch * m * n)
    s = ctx.stream()
    B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, out, stream=s)
    s.synchronize()
    with ctx.capture(s) as cap:
        B.lowrank_expand_device(ctx, batch, m, n, r, du, dx, dvt, out2, stream=s)
    assert cap.graph.launches == 1
    for _ in range(2):
        cap.graph.launch(s)
    s.synchronize()
    assert np.array_equal(out.download(), out2.download())
    assert np.array_equal(out.download(), O.lowrank_expand(batch, m, n, r, u, x, vt))
