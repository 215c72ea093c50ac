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


# ---- the analytic overlap schedule
def test_overlap_degenerate_threshold_is_serial(S):
    """threshold > total bytes -> one flush at the end; overlap time = serial time."""
    b, t = [3e6, 5e6, 2e6], [0.01, 0.02, 0.005]
    r = S.overlap_schedule(b, t, 1e9, 1e-4, 1e9, 4)
    assert len(r["buckets"]) == 1 and r["buckets"][0][0] == 2
    assert r["total_overlap"] == pytest.approx(r["total_serial"], rel=1e-12)
    assert r["total_serial"] == pytest.approx(0.035 + 1e-4 + 10e6 / 1e9 * 1.5, rel=1e-12)


def test_overlap_infinitely_fast_comm_hides_entirely(S):
    """bandwidth -> inf, latency 0 -> overlap time = the backward."""
    r = S.overlap_schedule([1e6] * 5, [0.1, 0.2, 0.3, 0.4, 0.5], 1.5e6, 0.0, 1e300, 8)
    assert r["total_overlap"] == pytest.approx(1.5, rel=1e-12)


def test_overlap_six_equal_layers_hand_trace(S):
    """6 equal layers, comm per layer = backward per layer, threshold = 1 layer -> backward + 1 comm slot.
    Hand-simulated event list: flush k (layer k) ready at k + 1, starts at once, ends at k + 2."""
    # W = 2: ring factor 2 (W-1)/W = 1, so 1e6 bytes at 1e6 B/s cost 1 s
    r = S.overlap_schedule([1e6] * 6, [1.0] * 6, 1e6, 0.0, 1e6, 2)
    assert [(k, rd, st, en) for k, rd, st, en in r["buckets"]] == [(k, k + 1.0, k + 1.0, k + 2.0) for k in range(6)]
    assert r["total_overlap"] == 7.0 and r["total_serial"] == 12.0


def test_overlap_slow_channel_queues_fifo(S):
    """Comm slower than the backward: flushes queue on the one channel.  Layers ready at 1, 2, 3; each
    flush costs 0.5 + 1.5 = 2 s -> starts 1, 3, 5, ends 3, 5, 7; serial = 3 + (0.5 + 4.5)."""
    r = S.overlap_schedule([1.0] * 3, [1.0] * 3, 0.0, 0.5, 1.0, 4)   # W = 4: ring factor 1.5
    ends = [e for _, _, _, e in r["buckets"]]
    starts = [s for _, _, s, _ in r["buckets"]]
    assert starts == pytest.approx([1.0, 3.0, 5.0]) and ends == pytest.approx([3.0, 5.0, 7.0])
    assert r["total_overlap"] == pytest.approx(7.0) and r["total_serial"] == pytest.approx(3.0 + 0.5 + 4.5)


def test_overlap_buckets_partition_layers_and_bound(S):
    """Random instances: flushes cover the layers in order (each closes at >= threshold, the last takes the rest),
    the channel never runs two flushes at once, and backward <= overlap <= serial + (flushes - 1) x latency."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        n = int(rng.integers(1, 40))
        b = rng.uniform(0, 5e6, n)
        t = rng.uniform(0, 2e-3, n)
        thr = float(rng.uniform(0, 2e7))
        lat, bw, W = float(rng.uniform(0, 5e-5)), float(rng.uniform(1e10, 1e12)), int(rng.integers(1, 9))
        r = S.overlap_schedule(b, t, thr, lat, bw, W)
        lasts = [k for k, *_ in r["buckets"]]
        assert lasts == sorted(lasts) and lasts[-1] == n - 1
        lo = 0
        for k in lasts[:-1]:
            assert b[lo:k + 1].sum() >= thr and (k == lo or b[lo:k].sum() < thr)
            lo = k + 1
        prev_end = 0.0
        for k, ready, start, end in r["buckets"]:
            assert ready == pytest.approx(t[:k + 1].sum()) and start >= max(ready, prev_end) - 1e-15
            prev_end = end
        assert t.sum() - 1e-12 <= r["total_overlap"] <= r["total_serial"] + len(lasts) * lat + 1e-12


def test_overlap_rejects_bad_arguments(S):
    with pytest.raises(ValueError):
        S.overlap_schedule([1.0], [1.0], -1.0, 0.0, 1.0, 2)
    with pytest.raises(ValueError):
        S.overlap_schedule([1.0], [1.0], 1.0, 0.0, 0.0, 2)
    with pytest.raises(ValueError):
        S.overlap_schedule([-1.0], [1.0], 1.0, 0.0, 1.0, 2)
