"""Straggler / batching side (PAPER.md 5), host-only native library libsmpu_sched.so.

Pins: SPEC S:268-272 / S:288-289 / S:318-319 / S:421-422 / S:440 examples and invariants, checked by brute force
in plain Python (partition, padded budget, contiguity in length order, least-squares recovery, idle fractions).
"""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def S():
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.exists(os.path.join(root, "paper_1806_00187_b200", "libsmpu_sched.so")):
        subprocess.run([sys.executable, os.path.join("paper_1806_00187_b200", "_build.py")], cwd=root, check=True)
    from paper_1806_00187_b200 import sched
    return sched


def corpus(n, seed=0):
    """WMT-like lengths: log-normal source (median ~24 tokens), target = source x U(0.67, 1.5) (P:278 ratio
    filter), both clipped to [1, 250] ("more than 250 words")."""
    rng = np.random.default_rng(seed)
    src = np.clip(np.round(rng.lognormal(np.log(24), 0.6, n)), 1, 250).astype(np.int32)
    tgt = np.clip(np.round(src * rng.uniform(0.67, 1.5, n)), 1, 250).astype(np.int32)
    return src, tgt


def batches(order, begin):
    return [order[begin[b]:begin[b + 1]] for b in range(len(begin) - 1)]


def key(src, tgt, i):
    return (max(src[i], tgt[i]), tgt[i], src[i], i)


def test_spec_token_budget_examples(S):
    src = tgt = np.full(4, 5)
    order, begin = S.token_budget(src, tgt, 20)            # budget 20 -> one sub-batch of 4
    assert [len(b) for b in batches(order, begin)] == [4]
    order, begin = S.token_budget(src, tgt, 10)            # budget 10 -> two sub-batches of 2
    assert [len(b) for b in batches(order, begin)] == [2, 2]
    with pytest.raises(ValueError):
        S.token_budget([300], [5], 100)                    # sentence longer than the budget


def test_token_budget_brute_force_validity(S):
    rng = np.random.default_rng(1)
    src = rng.integers(1, 101, 1000)
    tgt = rng.integers(1, 101, 1000)
    order, begin = S.token_budget(src, tgt, 3500)          # lengths uniform in [1,100], budget 3500
    bs = batches(order, begin)
    assert sorted(np.concatenate(bs).tolist()) == list(range(1000))               # partition
    for b in bs:                                                                    # padded budget
        assert len(b) * max(src[b].max(), tgt[b].max()) <= 3500
    ks = [key(src, tgt, i) for i in order]                                          # contiguity in sorted order
    assert ks == sorted(ks)
    # greedy maximality: adding the next sentence would have broken the budget
    for b, nxt in zip(bs[:-1], bs[1:]):
        j = nxt[0]
        assert (len(b) + 1) * max(src[b].max(), tgt[b].max(), src[j], tgt[j]) > 3500


def test_fit_timing_recovers_affine_and_degenerate_cases(S):
    rng = np.random.default_rng(2)
    sent = rng.integers(1, 200, 300)
    ms = rng.integers(1, 120, 300)
    mt = rng.integers(1, 120, 300)
    t = 3e-7 * sent * ms + 5e-7 * sent * mt + 2e-3                                   # exact affine cost
    assert np.allclose(S.fit_timing(sent, ms, mt, t), [3e-7, 5e-7, 2e-3], rtol=1e-6, atol=1e-12)
    c = S.fit_timing([10], [20], [30], [0.1])                                       # one measurement
    assert S.estimate([20], [30], [0], [0, 1], c)[0] == pytest.approx(0.1)
    c = S.fit_timing([10, 10], [20, 20], [30, 30], [0.1, 0.3])                      # mean of one bucket
    assert S.estimate([20], [30], [0], [0, 1], c)[0] == pytest.approx(0.2)
    # a negative fitted slope is clamped (monotone estimates)
    t2 = -1e-7 * sent * ms + 5e-7 * sent * mt + 2e-3
    c2 = S.fit_timing(sent, ms, mt, t2)
    assert c2[0] == 0 and c2[1] > 0


def test_time_balanced_batches(S):
    assert len(S.time_balanced([], [], [0, 0, 0.1], 0.1)[1]) == 1                  # empty corpus
    src, tgt = corpus(50)
    order, begin = S.time_balanced(src, tgt, [0, 0, 0.1], 0.1)                      # constant cost
    assert all(len(b) == 1 for b in batches(order, begin))
    src, tgt = corpus(20000, seed=3)
    coef = [3e-7, 5e-7, 2e-3]
    o1, b1 = S.token_budget(src, tgt, 3500)
    t1 = S.estimate(src, tgt, o1, b1, coef)
    target = np.percentile(t1, 90)                                                  # 90th percentile
    o2, b2 = S.time_balanced(src, tgt, coef, target)
    t2 = S.estimate(src, tgt, o2, b2, coef)
    assert sorted(o2.tolist()) == list(range(20000))
    assert np.all(t2[:-1] <= 1.1 * target * (1 + 1e-12))                            # overshoot cap
    cv = lambda t: t[:-1].std() / t[:-1].mean()  # noqa: E731  (the final remainder sub-batch excluded)
    assert cv(t2) < cv(t1)


def test_simulator(S):
    r = S.simulate(np.full(64, 0.11), 8, 2)                                         # equal times
    assert r["idle_fraction"] == 0 and r["steps"] == 4 and r["wall"] == pytest.approx(4 * 0.22)
    # a hand-traced case: W=2, c=1, times [1, 3, 2, 2] -> steps (max 3, idle 2) and (max 2, idle 0)
    r = S.simulate([1.0, 3.0, 2.0, 2.0], 2, 1)
    assert r["wall"] == 5.0 and r["idle_fraction"] == pytest.approx(2.0 / 10.0)
    src, tgt = corpus(200000, seed=4)
    o, b = S.token_budget(src, tgt, 3500)
    t = S.estimate(src, tgt, o, b, [3e-7, 5e-7, 2e-3])
    t = np.random.default_rng(5).permutation(t)                                     # shuffled sub-batches
    idle = [S.simulate(t, 8, c)["idle_fraction"] for c in (1, 2, 4, 8, 16)]
    assert idle[-1] < idle[0]                                                       # S:422 / P:179, Fig. 2
    assert all(a >= b - 1e-3 for a, b in zip(idle, idle[1:]))                      # S:440 (statistical)
