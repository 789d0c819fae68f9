"""GPU: the single-launch variable-size pointer-array kernel (lrb_varn.cu)
against the oracle's FMA chain, bitwise: ragged rows and columns (every
column count 1..71: whole fragments plus a zero-padded last one, several
64-column tiles, fewer than 8 columns), k tails, every op combination, beta = 1, padded leading dimensions,
repeated and graph-replayed executions (the self-resetting tile tickets), and
equality with the per-variant bucket path it replaced."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

OPS = [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")]


def _stored(op, r, c):
    return (c, r) if op == "T" else (r, c)


class PtrCase:
    def __init__(self, ctx, dims, opA="N", opB="N", beta=0.0, pad=0, seed=0, even_ld=True):
        rng = np.random.default_rng(seed)
        self.ctx, self.dims, self.opA, self.opB, self.beta = ctx, dims, opA, opB, beta
        self.ms = [d[0] for d in dims]
        self.ns = [d[1] for d in dims]
        self.ks = [d[2] for d in dims]
        self.hA, self.hB, self.hC0 = [], [], []
        self.lda, self.ldb, self.ldc = [], [], []
        self.dA, self.dB, self.dC = [], [], []
        for (m, n, k) in dims:
            sa, sb = _stored(opA, m, k), _stored(opB, k, n)
            la, lb, lc = max(1, sa[0]) + pad, max(1, sb[0]) + pad, max(1, m) + pad
            if even_ld:  # 16-byte leading dimensions: every operand TMA-addressable
                la, lb = la + (la & 1), lb + (lb & 1)
            a = rng.uniform(-1, 1, max(1, la * sa[1]))
            b = rng.uniform(-1, 1, max(1, lb * sb[1]))
            c = rng.uniform(-1, 1, max(1, lc * n)) if beta else np.full(max(1, lc * n), np.nan)
            self.hA.append(a)
            self.hB.append(b)
            self.hC0.append(c)
            self.lda.append(la)
            self.ldb.append(lb)
            self.ldc.append(lc)
            self.dA.append(ctx.to_device(a))
            self.dB.append(ctx.to_device(b))
            self.dC.append(ctx.to_device(c))

    def plan(self):
        return self.ctx.ptr_plan("C", self.opA, self.opB, self.ms, self.ns, self.ks, self.dA,
                                 self.lda, self.dB, self.ldb, self.dC, self.ldc, self.beta)

    def reset_c(self):
        for d, c in zip(self.dC, self.hC0):
            d.upload(c)

    def expect(self):
        out = [c.copy() for c in self.hC0]
        O.dgemm_ptr("C", self.opA, self.opB, self.ms, self.ns, self.ks, self.hA, self.lda,
                    self.hB, self.ldb, out, self.ldc, self.beta, threads=8)
        return out

    def check(self, expect=None):
        expect = expect or self.expect()
        for i, (d, e) in enumerate(zip(self.dC, expect)):
            got = d.download(e.size)
            assert np.array_equal(got, e, equal_nan=True), (
                f"item {i} {self.dims[i]}: max |diff| "
                f"{np.nanmax(np.abs(got - e)) if np.isfinite(got).all() else 'nan'}")


def _dims(seed, count=40, odd=False):
    """ragged shapes; even m and k keep every operand TMA-addressable (16-byte
    leading dimensions), odd ones send items to the bucket kernels too"""
    rng = np.random.default_rng(seed)
    dims = []
    ms = [1, 7, 64, 127, 128, 129, 200, 256, 300] if odd else [2, 8, 64, 126, 128, 130, 200, 256, 300]
    ks = [1, 3, 4, 13, 31, 32, 33, 64, 100, 257] if odd else [2, 4, 14, 30, 32, 34, 64, 100, 258]
    for _ in range(count):
        m = int(rng.choice(ms))
        n = int(rng.choice([1, 5, 8, 9, 15, 16, 23, 31, 33, 47, 56, 57, 63, 64, 65, 71, 100, 150]))
        k = int(rng.choice(ks))
        dims.append((m, n, k))
    return dims


@pytest.mark.parametrize("ops", OPS)
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_ragged_all_ops(ctx, ops, beta):
    c = PtrCase(ctx, _dims(sum(map(ord, ''.join(ops))) + int(beta)), ops[0], ops[1], beta, pad=0, seed=3)
    p = c.plan()
    assert p.launches == 1  # every item through the single launch
    p.execute()
    ctx.synchronize()
    c.check()


@pytest.mark.parametrize("ops", OPS)
def test_padded_leading_dimensions(ctx, ops):
    c = PtrCase(ctx, _dims(11, 24), ops[0], ops[1], 0.0, pad=6, seed=5)
    p = c.plan()
    assert p.launches == 1
    p.execute()
    ctx.synchronize()
    c.check()


@pytest.mark.parametrize("ops", OPS)
def test_odd_shapes_mix_single_launch_and_buckets(ctx, ops):
    c = PtrCase(ctx, _dims(17, 40, odd=True), ops[0], ops[1], 1.0, pad=1, seed=8, even_ld=False)
    p = c.plan()
    p.execute()
    ctx.synchronize()
    c.check()


@pytest.mark.parametrize("beta", [0.0, 1.0])
@pytest.mark.parametrize("ops", OPS)
def test_remainder_columns_every_width(ctx, beta, ops):
    # n = 8F + rem for every F in 0..8 and rem in 0..7, two row tiles, a k
    # tail: the last fragment column is zero-padded
    dims = [(150, n, 38) for n in range(1, 72)]
    c = PtrCase(ctx, dims, ops[0], ops[1], beta, seed=9)
    p = c.plan()
    assert p.launches == 1
    p.execute()
    ctx.synchronize()
    c.check()


def test_repeated_and_graph_replayed_executions(ctx):
    c = PtrCase(ctx, _dims(21, 60), seed=2)
    p = c.plan()
    exp = c.expect()
    s = ctx.stream()
    for _ in range(3):  # the tickets reset at the end of every launch
        c.reset_c()
        p.execute(s)
        s.synchronize()
        c.check(exp)
    with ctx.capture(s) as cap:
        p.execute(s)
    c.reset_c()
    for _ in range(3):
        cap.graph.launch(s)
    s.synchronize()
    c.check(exp)


def test_equals_the_bucket_path(ctx, monkeypatch):
    c = PtrCase(ctx, _dims(33, 50, odd=True), seed=4, even_ld=False)
    p = c.plan()
    p.execute()
    ctx.synchronize()
    one = [d.download(e.size) for d, e in zip(c.dC, c.hC0)]
    monkeypatch.setenv("LRB_PTR_BUCKETS", "1")
    c.reset_c()
    q = c.plan()
    assert q.launches > 1
    q.execute()
    ctx.synchronize()
    for d, a in zip(c.dC, one):
        assert np.array_equal(d.download(a.size), a, equal_nan=True)


def test_k_zero_and_empty_items_mixed_in(ctx):
    dims = [(64, 16, 0), (0, 8, 6), (34, 0, 8), (100, 40, 64), (6, 3, 2)]
    c = PtrCase(ctx, dims, seed=6)
    p = c.plan()
    p.execute()
    ctx.synchronize()
    c.check()
