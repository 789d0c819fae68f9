"""GPU against the reference's golden vectors (tests/golden/, produced by the
reference binary itself): the device result on the same inputs is bitwise the
FMA chain and inside BASELINE's componentwise bound of the reference output."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = np.load(os.path.join(HERE, "golden", "gemm_golden.npz"))
META = json.loads(bytes(GOLDEN["meta"]).decode())


def stored(order, op, r, c):
    s = (c, r) if op == "T" else (r, c)
    return s if order == "C" else (s[1], s[0])


def _device(ctx, order, opA, opB, m, n, k, batch, acc, A, B, C0):
    sa, sb, sc = stored(order, opA, m, k), stored(order, opB, k, n), stored(order, "N", m, n)
    out = C0.copy()
    ctx.dgemm_strided_batched_host(order, opA, opB, m, n, k, float(acc), A, sa[0], sa[0] * sa[1],
                                   B, sb[0], sb[0] * sb[1], out, sc[0], sc[0] * sc[1], batch)
    return out, sa, sb, sc


def _check(order, opA, opB, m, n, k, batch, acc, A, B, C0, got, want, sa, sb, sc):
    fma = C0.copy()
    O.dgemm_strided(order, opA, opB, m, n, k, float(acc), A, sa[0], sa[0] * sa[1], B, sb[0],
                    sb[0] * sb[1], fma, sc[0], sc[0] * sc[1], batch, threads=8)
    assert np.array_equal(got, fma)
    for it in range(batch):
        o = it * sc[0] * sc[1]
        bad, ratio = O.check_bound(order, opA, opB, m, n, k, float(acc), A[it * sa[0] * sa[1]:],
                                   sa[0], B[it * sb[0] * sb[1]:], sb[0], C0[o:] if acc else None,
                                   got[o:], want[o:], sc[0])
        assert bad == 0, f"item {it}: outside the FP64 bound (ratio {ratio})"


@pytest.mark.parametrize("case", META["small"], ids=[c[0] for c in META["small"]])
def test_device_vs_golden(ctx, case):
    name, order, opA, opB, m, n, k, batch, acc, seed = case
    A, B, C0 = GOLDEN[f"{name}__A"], GOLDEN[f"{name}__B"], GOLDEN[f"{name}__C0"]
    got, sa, sb, sc = _device(ctx, order, opA, opB, m, n, k, batch, acc, A, B, C0)
    _check(order, opA, opB, m, n, k, batch, acc, A, B, C0, got, GOLDEN[f"{name}__C"], sa, sb, sc)


@pytest.mark.parametrize("case", META["digest"], ids=[c[0] for c in META["digest"]])
def test_device_vs_golden_digest(ctx, case):
    name, order, opA, opB, m, n, k, batch, acc, seed, digest, first, last = case
    sa, sb, sc = stored(order, opA, m, k), stored(order, opB, k, n), stored(order, "N", m, n)
    A = O.fill_uniform(sa[0], sa[1], sa[0], sa[0] * sa[1], batch, seed, 0)
    B = O.fill_uniform(sb[0], sb[1], sb[0], sb[0] * sb[1], batch, seed, 1)
    C0 = np.zeros(sc[0] * sc[1] * batch)
    # the reference output, recomputed and authenticated by the golden digest
    want = C0.copy()
    O.dgemm_strided(order, opA, opB, m, n, k, 0.0, A, sa[0], sa[0] * sa[1], B, sb[0],
                    sb[0] * sb[1], want, sc[0], sc[0] * sc[1], batch, threads=8,
                    mode=O.REF_COMPILED)
    assert hashlib.sha256(want.tobytes()).hexdigest() == digest
    got, _, _, _ = _device(ctx, order, opA, opB, m, n, k, batch, acc, A, B, C0)
    _check(order, opA, opB, m, n, k, batch, acc, A, B, C0, got, want, sa, sb, sc)
