"""CPU: pin the oracle to the reference.

* golden vectors produced by the reference binary (tests/golden/make_golden.py,
  oracle/_ref built from /root/reference) — the C restatement must reproduce
  them BITWISE in its reference-rounding mode, and its FMA-chain mode (the
  device kernels' rounding) must sit inside BASELINE's componentwise bound;
* the reference's own known-answer cases (tests/test_core.cpp:24-49);
* the bound checker's negative control (tests/test_kernels.cpp:286-294);
* the counter RNG (host C == host Python, values pinned).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = np.load(os.path.join(HERE, "golden", "gemm_golden.npz"))
META = json.loads(bytes(GOLDEN["meta"]).decode())


def stored(order, op, r, c):
    s = (c, r) if op == "T" else (r, c)
    return s if order == "C" else (s[1], s[0])


def _inputs(order, opA, opB, m, n, k, batch, acc, seed):
    ar, ac = stored(order, opA, m, k)
    br, bc = stored(order, opB, k, n)
    cr, cc = stored(order, "N", m, n)
    A = O.fill_uniform(ar, ac, ar, ar * ac, batch, seed, 0)
    B = O.fill_uniform(br, bc, br, br * bc, batch, seed, 1)
    C0 = O.fill_uniform(cr, cc, cr, cr * cc, batch, seed, 2) if acc else np.zeros(cr * cc * batch)
    return A, B, C0, (ar, ac), (br, bc), (cr, cc)


def _oracle(mode, order, opA, opB, m, n, k, batch, acc, A, B, C0, sa, sb, sc):
    out = C0.copy()
    O.dgemm_strided(order, opA, opB, m, n, k, float(acc), A, sa[0], sa[0] * sa[1], B, sb[0],
                    sb[0] * sb[1], out, sc[0], sc[0] * sc[1], batch, threads=4, mode=mode)
    return out


@pytest.mark.parametrize("case", META["small"], ids=[c[0] for c in META["small"]])
def test_golden_small_cases(case):
    name, order, opA, opB, m, n, k, batch, acc, seed = case
    A, B, C0, sa, sb, sc = _inputs(order, opA, opB, m, n, k, batch, acc, seed)
    # the inputs the reference saw are exactly what the counter RNG regenerates
    assert np.array_equal(A, GOLDEN[f"{name}__A"])
    assert np.array_equal(B, GOLDEN[f"{name}__B"])
    assert np.array_equal(C0, GOLDEN[f"{name}__C0"])
    want = GOLDEN[f"{name}__C"]
    got = _oracle(O.REF_COMPILED, order, opA, opB, m, n, k, batch, acc, A, B, C0, sa, sb, sc)
    assert np.array_equal(got, want), "oracle restatement != reference binary"
    fma = _oracle(O.FMA_CHAIN, order, opA, opB, m, n, k, batch, acc, A, B, C0, sa, sb, sc)
    for it in range(batch):
        o = it * sc[0] * sc[1]
        bad, ratio = O.check_bound(order, opA, opB, m, n, k, float(acc), A[it * sa[0] * sa[1]:],
                                   sa[0], B[it * sb[0] * sb[1]:], sb[0],
                                   C0[o:] if acc else None, fma[o:], want[o:], sc[0])
        assert bad == 0, f"{name} item {it}: FMA chain outside the FP64 bound (ratio {ratio})"


@pytest.mark.parametrize("case", META["digest"], ids=[c[0] for c in META["digest"]])
def test_golden_baseline_digests(case):
    name, order, opA, opB, m, n, k, batch, acc, seed, digest, first, last = case
    A, B, C0, sa, sb, sc = _inputs(order, opA, opB, m, n, k, batch, acc, seed)
    got = _oracle(O.REF_COMPILED, order, opA, opB, m, n, k, batch, acc, A, B, C0, sa, sb, sc)
    assert got[0] == first and got[-1] == last
    assert hashlib.sha256(got.tobytes()).hexdigest() == digest


def test_golden_flops_counter():
    f = META["flops"]
    c = np.zeros(f["m"] * f["n"])
    fl = np.zeros(1, dtype=np.uint64)
    O.gemm_naive_raw(GOLDEN["flops__A"], GOLDEN["flops__B"], c, f["m"], f["k"], f["n"], False, fl)
    assert int(fl[0]) == f["count"] == 2 * f["m"] * f["n"] * f["k"]
    # the flops != NULL path is fully unfused in the reference binary
    assert np.array_equal(c, GOLDEN["flops__C"])


def test_known_answers_reference_tests():
    # tests/test_core.cpp:24-39
    ident = np.eye(3).ravel()
    mm = np.arange(1, 10, dtype=np.float64)
    c = np.zeros(9)
    O.gemm_naive_raw(ident, mm, c, 3, 3, 3, False)
    assert np.array_equal(c, mm)
    c = np.zeros(8)
    O.gemm_naive_raw(np.zeros(10), np.full(20, 3.25), c, 2, 5, 4, False)
    assert np.all(c == 0.0)
    c = np.zeros(4)
    O.gemm_naive_raw(np.array([1., 2, 3, 4]), np.array([5., 6, 7, 8]), c, 2, 2, 2, False)
    assert c.tolist() == [19, 22, 43, 50]
    # :41-49 accumulate
    c = np.full(4, 10.0)
    O.gemm_naive_raw(np.array([1., 0, 0, 1]), np.array([1., 2, 3, 4]), c, 2, 2, 2, True)
    assert c.tolist() == [11, 12, 13, 14]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 3, 4), (9, 7, 33), (31, 17, 64), (128, 16, 127)])
@pytest.mark.parametrize("acc", [False, True])
def test_restatement_equals_reference_binary(shape, acc):
    m, k, n = shape
    rng = np.random.default_rng(m * 100 + k)
    a, b = rng.uniform(-1, 1, m * k), rng.uniform(-1, 1, k * n)
    c0 = rng.uniform(-1, 1, m * n)
    for with_flops in (False, True):
        c1, c2 = c0.copy(), c0.copy()
        f1 = np.zeros(1, np.uint64) if with_flops else None
        f2 = np.zeros(1, np.uint64) if with_flops else None
        O.ref_gemm_naive_raw(a, b, c1, m, k, n, acc, f1)
        O.gemm_naive_raw(a, b, c2, m, k, n, acc, f2)
        assert np.array_equal(c1, c2)
        if with_flops:
            assert f1[0] == f2[0] == 2 * m * n * k


def test_bound_checker_negative_control():
    m, n, k = 12, 6, 10
    A = O.fill_uniform(m, k, m, m * k, 1, 7, 0)
    B = O.fill_uniform(k, n, k, k * n, 1, 7, 1)
    ref = np.zeros(m * n)
    O.dgemm_strided("C", "N", "N", m, n, k, 0.0, A, m, 0, B, k, 0, ref, m, 0, 1,
                    mode=O.REF_COMPILED)
    good = np.zeros(m * n)
    O.dgemm_strided("C", "N", "N", m, n, k, 0.0, A, m, 0, B, k, 0, good, m, 0, 1)
    assert O.check_bound("C", "N", "N", m, n, k, 0.0, A, m, B, k, None, good, ref, m)[0] == 0
    bad = good.copy()
    bad[5] += 1e-9
    nbad, ratio = O.check_bound("C", "N", "N", m, n, k, 0.0, A, m, B, k, None, bad, ref, m)
    assert nbad == 1 and ratio > 1.0
    nan = good.copy()
    nan[3] = np.nan
    assert O.check_bound("C", "N", "N", m, n, k, 0.0, A, m, B, k, None, nan, ref, m)[0] == 1


def test_rng_c_matches_python_and_is_pinned():
    x = O.fill_uniform(5, 3, 7, 21, 2, 9, 1, 100)
    key = W.stream_key(9, 1)
    for it in range(2):
        for c in range(3):
            for r in range(5):
                assert x[it * 21 + c * 7 + r] == W.uniform(key, 100 + it, r + c * 5)
    # pinned values (a change of generator breaks every stored golden vector)
    assert W.uniform(W.stream_key(0, 0), 0, 0) == O.fill_uniform(1, 1, 1, 1, 1, 0, 0)[0]
    v = O.fill_uniform(1000, 1, 1000, 1000, 1, 3, 0)
    assert v.min() >= -1.0 and v.max() < 1.0 and abs(v.mean()) < 0.1


def test_cfg4_shapes_are_deterministic():
    w = W.get("cfg4")
    assert len(w.bs) == 8192 and set(w.bs) == {256, 512, 1024}
    assert min(w.rs) == 8 and max(w.rs) == 64
    w2 = W.Variable("cfg4", 8192, seed=3)
    assert w.bs == w2.bs and w.rs == w2.rs
    assert 29.0 < w.bytes() / 2 ** 30 < 32.0  # ~30.6 GiB


# ------------------------------------------------ the paper's low-rank product
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("batch,block,rank", [(3, 16, 4), (7, 17, 3), (5, 256, 8), (4, 512, 16),
                                              (2, 64, 32), (3, 1, 1), (2, 33, 40)])
def test_lowrank_restatement_equals_reference_binary(batch, block, rank):
    # the reference's own naive_multiply_batch (bench.hpp:55-77 -> low_rank.hpp:73-87)
    from paper_2311_07602_b200 import lowrank as L

    b = L.LowRankBatch.random(batch, block, rank, batch * 100 + rank)
    args = (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
    want = O.ref_lowrank(0, batch, block, rank, *args, workers=2)
    got = O.lowrank(batch, block, rank, *args, threads=2, mode=O.REF_COMPILED)
    assert np.array_equal(got, want)
    fma = O.lowrank(batch, block, rank, *args, threads=2)
    bad, ratio = O.lowrank_bound_check(batch, block, rank, *args, fma, want)
    assert bad == 0
    err, _, _ = O.ref_compare_to_reference(batch, block, rank, *args, fma)
    assert err < 1e-12
    # the reference's fused and packed drivers agree with its oracle to its own tolerance
    for which in (1, 2):  # packed: the reference's plan (live or tests/golden/packing_plans.json)
        other = O.ref_lowrank(which, batch, block, rank, *args, workers=2)
        assert O.ref_compare_to_reference(batch, block, rank, *args, other)[0] < 1e-11


def test_lowrank_flops_accounting():
    from paper_2311_07602_b200 import lowrank as L
    from paper_2311_07602_b200._lib import lib

    # tests/test_core.cpp:95-99
    for r, b, want in ((8, 512, 67584), (1, 1, 6), (32, 2048, 4325376)):
        assert L.flops_per_item(r, b) == want == lib.lrb_lowrank_flops_per_item(r, b)


def test_packing_plan_fixture_matches_the_reference():
    # tests/golden/packing_plans.json replays make_packing_plan where the
    # machine files are absent (the GPU box); pin it against the live call
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "packing_plans.json")
    fx = json.load(open(path))
    assert fx["fields"] == list(O.PLAN_FIELDS)
    assert all(fx["plans"][O.DEFAULT_MACHINE][str(r)] is not None for r in range(1, 129))
    if not (O.ref_available() and O.ref_machines_available()):
        pytest.skip("the reference's machine files are not here")
    for m, plans in fx["plans"].items():
        for r in (1, 7, 8, 16, 31, 64, 128):
            assert O.ref_packing_plan_live(m, r) == plans[str(r)], (m, r)


def test_packed_drivers_replay_the_fixture_plan(monkeypatch):
    # what the GPU box does: packed_multiply / blr_matvec with the committed plan
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2311_07602_b200 import lowrank as L

    b = L.LowRankBatch.random(5, 64, 8, 77)
    args = (b.a_vt_batch, b.b_u_batch, b.a_x_batch, b.b_x_batch)
    live = O.ref_lowrank(2, 5, 64, 8, *args, workers=2) if O.ref_machines_available() else None
    monkeypatch.setattr(O, "ref_machines_available", lambda: False)
    replay = O.ref_lowrank(2, 5, 64, 8, *args, workers=2)
    assert O.ref_compare_to_reference(5, 64, 8, *args, replay)[0] < 1e-11
    if live is not None:
        assert np.array_equal(live, replay)


@pytest.mark.parametrize("batch,m,n,r", [(3, 17, 13, 5), (2, 64, 64, 8), (1, 33, 40, 33),
                                         (2, 9, 9, 1)])
def test_expand_restatement_equals_reference_binary(batch, m, n, r):
    # dense_gemm_naive(dense_gemm_naive(U, X), Vt) per item (blr.hpp:75-78)
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(batch * 100 + m + r)
    u, x, vt = (rng.uniform(-1, 1, s) for s in (batch * m * r, batch * r * r, batch * r * n))
    want = O.ref_lowrank_expand(batch, m, n, r, u, x, vt)
    assert np.array_equal(O.lowrank_expand(batch, m, n, r, u, x, vt, mode=O.REF_COMPILED), want)


@pytest.mark.parametrize("n,block,rank", [(96, 32, 6), (40, 8, 3), (64, 64, 4)])
def test_reconstruct_restatement_equals_reference_binary(n, block, rank):
    # BlrMatrix::reconstruct_dense (blr.hpp:62-86)
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2311_07602_b200 import blr as B

    m = B.BlrMatrix.random(n, block, rank, n + block)
    args = (n, block, rank) + m.packed_arrays()
    assert np.array_equal(O.blr_reconstruct(*args, mode=O.REF_COMPILED),
                          O.ref_blr_reconstruct(*args))
