"""The exact early overflow decision of the W > 1 path (csrc/kernels.cuh K0 EARLY), checked on CPU as
arithmetic: from the per-rank max magnitudes M_r of the accumulated fp16 gradients A_r alone,
  * some A_r non-finite          => R = rn16 fold of A_0 .. A_{W-1} is non-finite (NaN / inf propagate), and
  * sum_r M_r <= 2^15, all finite => R is finite for ANY values bounded by the M_r, in ascending-rank order with an
    rn16 after each add (reading R3) -- every partial sum stays below 65520, the first value that rounds to inf;
otherwise the decision is deferred to the sweep of R.  numpy's float16 adds round to nearest even (pinned against
the oracle's own binary16 codec in tests/test_oracle.py)."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

F16_MAX_FINITE_SUM = 65520.0      # the smallest real that rounds to +inf in binary16


def fold(rows):
    acc = rows[0].astype(np.float16)
    for r in rows[1:]:
        acc = (acc + r.astype(np.float16)).astype(np.float16)
    return acc


@settings(max_examples=300, deadline=None)
@given(st.integers(2, 8), st.integers(0, 2 ** 31 - 1), st.booleans())
def test_sum_of_maxima_within_2_15_never_overflows(W, seed, adversarial):
    rng = np.random.default_rng(seed)
    # split the budget 2^15 among the ranks, then draw values bounded by each rank's maximum
    share = rng.dirichlet(np.ones(W)) * 32768.0
    rows = []
    for m in share:
        m16 = np.float16(m)
        if np.float16(m16) > m:                        # round the bound down to an fp16 value <= m
            m16 = np.nextafter(m16, np.float16(0))
        n = 64
        if adversarial:                                # same sign, at the bound: the largest partial sums
            x = np.full(n, m16, np.float16)
        else:
            x = (rng.uniform(-1, 1, n) * float(m16)).astype(np.float16)
            x = np.clip(x, -m16, m16)
        rows.append(x)
    assert sum(float(np.abs(r).max()) for r in rows) <= 32768.0
    R = fold(rows)
    assert np.isfinite(R).all()
    # and every partial sum stays below the rounding-to-inf threshold
    acc = rows[0].astype(np.float64)
    for r in rows[1:]:
        acc = np.float16(acc + r).astype(np.float64)
        assert (np.abs(acc) < F16_MAX_FINITE_SUM).all()


@settings(max_examples=200, deadline=None)
@given(st.integers(2, 8), st.integers(0, 2 ** 31 - 1), st.sampled_from([np.inf, -np.inf, np.nan]))
def test_a_non_finite_rank_makes_R_non_finite(W, seed, bad):
    rng = np.random.default_rng(seed)
    rows = [(rng.standard_normal(32) * 100).astype(np.float16) for _ in range(W)]
    r, i = int(rng.integers(0, W)), int(rng.integers(0, 32))
    rows[r][i] = bad
    R = fold(rows)
    assert not np.isfinite(R[i])


def test_the_bound_is_needed():
    """Above the budget a fold can overflow with every A_r finite (RED_OVF: 40000 + 40000), which is why the
    decision then waits for the sweep of R instead of calling it clean."""
    rows = [np.array([40000.0], np.float16), np.array([40000.0], np.float16)]
    assert all(np.isfinite(r).all() for r in rows) and np.isinf(fold(rows)).all()
    assert np.isinf(np.float16(65520.0)) and np.isfinite(np.float16(65519.0))
