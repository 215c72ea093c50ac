"""Randomised W > 1 parity over virtual ranks (hypothesis, fixed seed): random tensor lists (1..40k elements, every
class), W = 2..8, update_freq 1..4, bucket thresholds from a few bytes to 1 MiB, the SM or copy-engine bucket
all-reduce (ar_copy_engine 0 / 1 / 2), ar_pieces 1..3, the replicated or sharded layout, every way of interleaving
the ranks' calls (micro-batch by micro-batch, rank-major, last micro-batch bucket-wise in random rank x bucket order,
resident accumulate_many), injected non-finites on any rank and micro-batch, RED_OVF (finite everywhere, overflow
only in the sum) and BIG (a finite 40000 after the sum: the early decision must defer to the sweep); the library vs
the oracle (ascending-rank rn16 reduce, reading R3) on decisions and R (bitwise) and theta/m/v/w16 (tolerance),
every update, replicas identical; the fp32 accumulator (Z1) and
split-tensor buckets in a quarter of the cases each; 200 cases (~12 s)."""
import hashlib

import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, seed, settings
from hypothesis import strategies as st

import oracle as O
import synth
from synth import models
from tests.gpu_util import (Magnitudes, check_state, decisions, format_report, gpu_state, lib_cfg, oracle_decisions,
                            rtol_for, snapshot, ulp16_dist)
from tests.test_gpu_virtual import _feed, _same_r

pytestmark = pytest.mark.gpu
REPORT = []


@st.composite
def cases(draw):
    nt = draw(st.integers(1, 5))
    tensors = [(f"t{j}", draw(st.integers(1, 40_000)), draw(st.integers(0, 2))) for j in range(nt)]
    n = sum(t[1] for t in tensors)
    W = draw(st.integers(2, 8))
    c = draw(st.integers(1, 4))
    inj = []
    for u in (1, 2, 3):
        if draw(st.integers(0, 3)) == 0:
            kind = draw(st.sampled_from(["INF", "NINF", "NAN", "RED_OVF", "BIG"] + (["ACC_OVF"] if c >= 2 else [])))
            d = dict(u=u, kind=kind, i=draw(st.integers(0, n - 1)))
            if kind in ("INF", "NINF", "NAN"):
                d.update(r=draw(st.integers(0, W - 1)), k=draw(st.integers(1, c)))
            elif kind == "ACC_OVF":
                d.update(r=draw(st.integers(0, W - 1)))
            inj.append(d)
    sharded = draw(st.booleans())
    ce = 0 if sharded else draw(st.integers(0, 2))
    pieces = 1 if sharded else draw(st.integers(1, 3))
    mode = draw(st.sampled_from(["calls", "rank_major", "buckets", "many"]))
    bucket_bytes = draw(st.sampled_from([2, 1000, 16_384, 100_000, 1 << 20]))
    acc32 = draw(st.integers(0, 3)) == 0          # SURVEY Z1's fp32 accumulator in a quarter of the cases
    split = draw(st.integers(0, 3)) == 0          # split_tensors: buckets cut through tensors
    return tensors, W, c, inj, sharded, ce, pieces, mode, bucket_bytes, draw(st.integers(0, 1000)), acc32, split


@seed(int(os.environ.get("SMPU_FUZZ_SEED", 20261019)))
@settings(max_examples=int(os.environ.get("SMPU_FUZZ_EXAMPLES", 200)), deadline=None,
          suppress_health_check=list(HealthCheck))
@given(cases())
def test_virtual_fuzz_against_oracle(case):
    import paper_1806_00187_b200 as P
    tensors, W, c, inj, sharded, ce, pieces, mode, bucket_bytes, order_seed, acc32, split = case
    if mode == "many" and c == 1:
        mode = "calls"
    wl = models.Workload("vfuzz", tensors, W, c, injections=inj)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    ocfg = O.Config(accum_fp32=acc32)
    grp = P.VirtualGroup(wl.numel, theta0, lib_cfg(wl, ocfg, bucket_bytes=bucket_bytes, sharded=int(sharded),
                                                   ar_copy_engine=ce, ar_pieces=pieces, split_tensors=int(split)),
                         world=W)
    ms = grp.members
    bb = ms[0].bucket_begin
    ranges = [m.shard_ranges() for m in ms]
    orc = O.Oracle(theta0, ocfg)
    mags = Magnitudes(theta0)
    rng = np.random.default_rng(order_seed)
    import tests.test_gpu_virtual as V
    saved_c = V.C
    V.C = c                                   # _feed's micro-batch count
    try:
        for u in range(1, 4):
            e = orc.e
            grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, e) for k in range(1, c + 1)] for r in range(W)]
            toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(W)]
            if mode == "many":                # accumulate_many over all c on every rank
                for r in range(W):
                    ms[r].accumulate_many([V.h2t(x) for x in grads[r]], toks[r])
            else:
                _feed(ms, grads, toks, mode, rng, bb)
            for r in rng.permutation(W):
                ms[r].step(wait=False)
            res = [m.result(u) for m in ms]
            before = snapshot(orc)
            ores = orc.update(grads, toks)
            for r in range(W):
                assert decisions(res[r]) == oracle_decisions(ores), (case, u, r)
            if ores["applied"]:
                mags.update(ores["R"], ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
            for r in range(W):
                acc = ms[r].get_state(P.smpu.STATE_ACCUM)
                spans = ranges[r] if sharded else [(0, lay.n)]
                assert all(_same_r(acc, ores["R"], lo, hi) for lo, hi in spans), (case, u, r, "R")
            states = [gpu_state(m) for m in ms]
            w16 = states[0]["w16"]
            assert all(np.array_equal(s["w16"], w16) for s in states), (case, u, "w16 replicas")
            rtol = rtol_for(orc.s.t)
            if sharded:
                for r in range(W):
                    if not ranges[r]:
                        continue
                    idx = np.concatenate([np.arange(lo, hi) for lo, hi in ranges[r]])
                    if idx.size == 0:
                        continue
                    got = {k: v[idx] for k, v in states[r].items()}
                    sub = type(mags).__new__(type(mags))
                    sub.th, sub.m, sub.th1, sub.m1 = mags.th[idx], mags.m[idx], mags.th1[idx], mags.m1[idx]
                    check_state(got, snapshot(orc, idx), sub, rtol, where=f"{case} u{u} r{r}", report=REPORT)
                assert ulp16_dist(w16, orc.w16).max() <= 1, (case, u)
            else:
                h = {hashlib.sha256(b"".join(s[x].tobytes() for x in ("theta", "m", "v", "w16"))).hexdigest()
                     for s in states}
                assert len(h) == 1, (case, u, "replicas differ")
                check_state(states[0], snapshot(orc), mags, rtol, where=f"{case} u{u}", report=REPORT)
    finally:
        V.C = saved_c
        grp.close()


def test_virtual_fuzz_error_report():
    if not REPORT:
        pytest.skip("the fuzz test did not run")
    print("virtual fuzz worst errors:", format_report(REPORT))
