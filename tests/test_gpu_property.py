"""Property-based parity (hypothesis): random orders, ops, shapes (ragged,
tiny, k = 0), beta, batch sizes, leading-dimension and item padding — every
draw through lrb_dgemm_strided_batched with the automatic selector (so the
m/n/k rules, the k64 tiles, s96/t64 and the TMA-store epilogue all get hit),
checked bitwise against the FMA-chain oracle with NaN-poisoned gaps and
within BASELINE's bound against the reference rounding."""
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from helpers import Case  # noqa: E402

pytestmark = pytest.mark.gpu

dims = st.sampled_from([1, 2, 3, 7, 8, 13, 16, 24, 31, 32, 33, 48, 64, 65, 96, 100, 128, 130, 200])
ks = st.sampled_from([0, 1, 3, 4, 8, 13, 16, 17, 32, 40, 64, 96, 128, 257])


@settings(max_examples=120, deadline=None,
          suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(order=st.sampled_from(["C", "R"]), opA=st.sampled_from(["N", "T"]),
       opB=st.sampled_from(["N", "T"]), m=dims, n=dims, k=ks,
       batch=st.integers(min_value=1, max_value=5), beta=st.sampled_from([0.0, 1.0]),
       pad=st.tuples(*[st.integers(0, 6)] * 3), spad=st.tuples(*[st.integers(0, 9)] * 3),
       seed=st.integers(0, 2 ** 16))
def test_random_strided_batches_match_the_oracle(ctx, order, opA, opB, m, n, k, batch, beta, pad,
                                                 spad, seed):
    c = Case(order, opA, opB, m, n, k, batch, beta=beta, pad=pad, spad=spad, seed=seed)
    c.check(c.run_device(ctx))


panel_rows = st.sampled_from([1, 8, 100, 128, 129, 200, 255, 256, 257, 300, 384, 512, 520])
panel_cols = st.sampled_from([1, 7, 31, 32, 33, 64, 95, 96, 100, 160, 257])
panel_ks = st.integers(min_value=1, max_value=32)


@settings(max_examples=80, deadline=None,
          suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(order=st.sampled_from(["C", "R"]), opX=st.sampled_from(["N", "T"]), rows=panel_rows,
       cols=panel_cols, k=panel_ks, batch=st.integers(min_value=1, max_value=4),
       beta=st.sampled_from([0.0, 1.0]), pad=st.tuples(*[st.integers(0, 3)] * 3),
       spad=st.tuples(*[st.integers(0, 5)] * 3), seed=st.integers(0, 2 ** 16))
def test_random_panel_kernel_batches_match_the_oracle(ctx, order, opX, rows, cols, k, batch, beta,
                                                      pad, spad, seed):
    # the row-panel kernel forced (p256): ragged 256-row units and 32-column
    # chunks, every k in 1..32, both B layouts, row-major calls; operands TMA
    # cannot address fall back to the tile kernel, and both must be exact
    if order == "C":
        c = Case("C", "N", opX, rows, cols, k, batch, beta=beta, pad=pad, spad=spad, seed=seed)
    else:  # row-major C = op(A) op(B) is column-major C^T: panel when op(B) = N
        c = Case("R", opX, "N", cols, rows, k, batch, beta=beta, pad=pad, spad=spad, seed=seed)
    c.check(c.run_device(ctx, "p256"))
