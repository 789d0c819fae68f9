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
