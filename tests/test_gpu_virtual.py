"""The world > 1 path on ONE GPU: W virtual ranks (smpu_group_init) against the oracle, bitwise.

Every peer kernel of the multi-GPU path -- the fused bucket all-reduce, the exact early
overflow decision exchange and the late sweep decision (readings R3/R4), the sharded reduce-scatter + Adam
+ w16 all-gather -- is the same template instantiated over local windows (csrc/lsa_allreduce.cuh,
LocalPeers), so these tests execute the W = 2..8 arithmetic on the driver's one-GPU box: SURVEY rows a5, a6, f1, f2.

Inputs: ragged tensors whose buckets (400 kB threshold) start and end off the 8/16-element vector grid, G_real
(order-sensitive values: bitwise parity holds because the fused sum is the oracle's ascending-rank order) and
G_exact, with every injection kind: RED_OVF (finite A_r, inf only after the sum: early decision undecided -> sweep
-> skip), BIG (a finite 40000 after the sum: undecided -> sweep -> late apply), INF (a non-finite A_r: early
skip), ACC_OVF (65504 + 65504 inside one rank: early skip).
"""
import hashlib

import numpy as np
import pytest

import oracle as O
import synth
from synth import models
from tests.gpu_util import (Magnitudes, check_state, decisions, format_report, gpu_state, h2t, lib_cfg,
                            oracle_decisions, rtol_for, snapshot, ulp16_dist)

pytestmark = pytest.mark.gpu

TENSORS = [("w0", 300_001, 0), ("b0", 1025, 1), ("w1", 262_144, 0), ("e", 131_072, 2), ("b1", 7, 1)]
C = 3


def _workload(world, family, updates):
    inj = [dict(u=3, kind="RED_OVF", i=262_150), dict(u=4, kind="BIG", i=300_500),
           dict(u=5, kind="INF", r=world - 1, k=2, i=17), dict(u=6, kind="ACC_OVF", r=0, i=400_000)]
    return models.Workload("virtual", TENSORS, world, C, injections=[x for x in inj if x["u"] <= updates],
                           family=family)


def _same_r(got, ref, lo=0, hi=None):
    g, r = got[lo:hi], ref[lo:hi]
    nan = np.isnan(r.view(np.float16))
    return np.array_equal(np.isnan(g.view(np.float16)), nan) and np.array_equal(g[~nan], r[~nan])


def _feed(members, grads, toks, mode, rng, bb):
    """Give every rank its c micro-batches, interleaving the ranks' calls the way `mode` says."""
    W = len(members)
    if mode == "calls":                      # micro-batch by micro-batch, ranks in order
        for k in range(C):
            for r in range(W):
                members[r].accumulate(h2t(grads[r][k]), toks[r][k])
    elif mode == "rank_major":               # rank by rank (the last rank's last call issues every collective)
        for r in reversed(range(W)):
            for k in range(C):
                members[r].accumulate(h2t(grads[r][k]), toks[r][k])
    elif mode == "buckets":                  # last micro-batch bucket-wise, buckets and ranks in random order
        for k in range(C - 1):
            for r in range(W):
                members[r].accumulate(h2t(grads[r][k]), toks[r][k])
        for r in range(W):
            members[r].micro_begin(toks[r][C - 1])
        todo = [(r, b) for r in range(W) for b in range(len(bb) - 1)]
        rng.shuffle(todo)
        for r, b in todo:
            members[r].accumulate_bucket(b, h2t(grads[r][C - 1][bb[b]:bb[b + 1]]))
    elif mode == "many":                     # resident micro-batches: the final one inside accumulate_many
        for r in range(W):
            members[r].accumulate(h2t(grads[r][0]), toks[r][0])
            members[r].accumulate_many([h2t(x) for x in grads[r][1:]], toks[r][1:])
    else:
        raise ValueError(mode)


def _run(world, family="real", sharded=False, mode="calls", updates=6, acc32=False, **cfg_kw):
    import paper_1806_00187_b200 as P
    wl = _workload(world, family, updates)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    cfg_kw.setdefault("bucket_bytes", 400_000)
    ocfg = O.Config(accum_fp32=acc32)
    grp = P.VirtualGroup(wl.numel, theta0, lib_cfg(wl, ocfg, sharded=int(sharded), **cfg_kw), world=world)
    members = grp.members
    bb = members[0].bucket_begin
    assert len(bb) - 1 >= 2 and any(int(x) % 16 for x in bb[1:-1]), "buckets must cut off the vector grid"
    ranges = [m.shard_ranges() for m in members]
    if sharded:
        mark = np.zeros(lay.n, np.int32)
        for rr in ranges:
            for lo, hi in rr:
                mark[lo:hi] += 1
        assert (mark == 1).all(), "shards must partition the vector"
    orc = O.Oracle(theta0, ocfg)
    mags = Magnitudes(theta0)
    rng = np.random.default_rng(world * 131 + len(mode))
    report, seen = [], set()
    e = 7
    for u in range(1, updates + 1):
        grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, e) for k in range(1, C + 1)] for r in range(world)]
        toks = [[synth.ntokens(wl, u, r, k) for k in range(1, C + 1)] for r in range(world)]
        _feed(members, grads, toks, mode, rng, bb)
        for r in rng.permutation(world):
            members[r].step(wait=False)
        res = [m.result(u) for m in members]
        before = snapshot(orc)
        ores = orc.update(grads, toks)
        seen.add((ores["overflow"], ores["applied"]))
        for r in range(world):
            assert decisions(res[r]) == oracle_decisions(ores), (u, r, decisions(res[r]), oracle_decisions(ores))
        if ores["applied"]:
            mags.update(ores["R"], ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
        # the reduced gradient R, bitwise (NaN as a class): everywhere (replicated) or on the rank's shard
        for r in range(world):
            acc = members[r].get_state(P.smpu.STATE_ACCUM)
            spans = ranges[r] if sharded else [(0, lay.n)]
            assert all(_same_r(acc, ores["R"], lo, hi) for lo, hi in spans), f"update {u} rank {r}: R differs"
        states = [gpu_state(m) for m in members]
        w16 = states[0]["w16"]
        assert all(np.array_equal(s["w16"], w16) for s in states), f"update {u}: replicas' w16 differ"
        rtol = rtol_for(orc.s.t)
        if sharded:
            for r in range(world):
                idx = np.concatenate([np.arange(lo, hi) for lo, hi in ranges[r]])
                got = {k: v[idx] for k, v in states[r].items()}
                sub = type(mags).__new__(type(mags))
                sub.th, sub.m, sub.th1, sub.m1 = mags.th[idx], mags.m[idx], mags.th1[idx], mags.m1[idx]
                check_state(got, snapshot(orc, idx), sub, rtol, where=f"update {u} rank {r} shard", report=report)
            d = ulp16_dist(w16, orc.w16)        # the all-gathered w16: every element, every replica
            assert d.max() <= 1, f"update {u}: w16 differs by {d.max()} ulp"
        else:
            h = [hashlib.sha256(b"".join(s[x].tobytes() for x in ("theta", "m", "v", "w16"))).hexdigest()
                 for s in states]
            assert len(set(h)) == 1, f"update {u}: replicas differ"
            check_state(states[0], snapshot(orc), mags, rtol, where=f"update {u}", report=report)
        e = res[0]["scale_log2_next"]
    grp.close()
    if updates >= 6:
        assert (1, 0) in seen and (0, 1) in seen
    print(f"virtual W={world} {family} {'sharded' if sharded else 'replicated'} {mode}: {format_report(report)}")


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("sharded", [False, True], ids=["replicated", "sharded"])
def test_virtual_world_bitwise(world, sharded):
    """G_real, call by call: decisions and R bitwise, theta/m/v within c.4 (1e-6 at update 1), w16 <= 1 ulp,
    replicas identical; through RED_OVF / BIG / INF / ACC_OVF."""
    _run(world, "real", sharded)


@pytest.mark.parametrize("world,sharded", [(3, False), (8, True), (5, False)])
def test_virtual_buckets_out_of_order(world, sharded):
    """Bucket-wise last micro-batches, buckets and ranks interleaved at random: all-reduces still issue in canonical
    bucket order and R is unchanged."""
    _run(world, "real", sharded, mode="buckets")


@pytest.mark.parametrize("world,split", [(4, 5), (2, 3)])
def test_virtual_pieces(world, split):
    """smpu_config.ar_pieces: every bucket all-reduced as `split` pieces, Adam of each right behind it; same bits
    as one launch per bucket (the oracle's)."""
    _run(world, "real", False, mode="buckets", ar_pieces=split)


@pytest.mark.parametrize("world,mode,split,ce", [(2, "calls", 1, 1), (3, "buckets", 1, 1), (4, "calls", 3, 1),
                                                 (8, "buckets", 1, 1), (5, "many", 2, 1), (4, "buckets", 1, 2),
                                                 (8, "calls", 2, 2)])
def test_virtual_copy_engine(world, mode, split, ce):
    """smpu_config.ar_copy_engine: the bucket all-reduce's traffic moved by cudaMemcpyAsync (push of every shard to
    its owner's staging, fold, all-gather of R): decisions and R bitwise the oracle's (the fold is k_ar32's
    ascending-rank order), alone and with ar_pieces, through every injection kind; ce = 2: every bucket but the last
    on the copy engines, the last through k_ar32 (the two share the LSA barriers)."""
    _run(world, "real", False, mode=mode, ar_copy_engine=ce, ar_pieces=split)


@pytest.mark.parametrize("world,ce,sharded", [(3, 0, False), (8, 1, False), (5, 2, False), (6, 0, True)])
def test_virtual_one_bucket_per_tensor(world, ce, sharded):
    """bucket_bytes = 2: every tensor its own bucket, down to the 7-element bias -- buckets with no whole 16-element
    unit (the fold is all head / tail, the copy engines move nothing), shards empty on most ranks; SM, copy-engine
    and copy-engine-but-last all-reduces and the sharded layout, bitwise against the oracle."""
    _run(world, "real", sharded, mode="calls", bucket_bytes=2, ar_copy_engine=ce)


@pytest.mark.parametrize("world,c,ce,sharded", [(2, 1, 0, False), (3, 2, 1, False), (4, 3, 0, True), (2, 1, 0, True)])
def test_virtual_nonfinite_in_bucket_head_and_tail(world, c, ce, sharded):
    """A non-finite in the ragged head or tail of a bucket, handled by a thread that also accumulated a 16-element
    vector unit: the max |A_r| statistic of the early decision must still see it (regression: the element path once
    took a scalar max against the two packed lanes of the vector path's max, so an INF at a bucket's first elements
    was lost and the update applied).  Buckets of one tensor each: [0, 1), [1, 32), [32, 1032), [1032, 1065);
    INF at 1 (head of bucket 1), NaN at 1031 (tail of bucket 2), -INF at 1064 (tail of the last), each on one rank
    and micro-batch, then a clean update; decisions and R bitwise the oracle's."""
    import paper_1806_00187_b200 as P
    tensors = [("a", 1, 0), ("b", 31, 0), ("c", 1000, 1), ("d", 33, 2)]
    inj = [dict(u=1, kind="INF", r=0, k=1, i=1), dict(u=2, kind="NAN", r=world - 1, k=c, i=1031),
           dict(u=3, kind="NINF", r=world // 2, k=1, i=1064)]
    wl = models.Workload("headtail", tensors, world, c, injections=inj)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    grp = P.VirtualGroup(wl.numel, theta0, lib_cfg(wl, bucket_bytes=2, sharded=int(sharded), ar_copy_engine=ce),
                         world=world)
    ms = grp.members
    assert list(ms[0].bucket_begin) == [0, 1, 32, 1032, 1065]
    orc = O.Oracle(theta0)
    for u in range(1, 5):
        grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, orc.e) for k in range(1, c + 1)] for r in range(world)]
        toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(world)]
        for k in range(c):
            for r in range(world):
                ms[r].accumulate(h2t(grads[r][k]), toks[r][k])
        for m in ms:
            m.step(wait=False)
        ores = orc.update(grads, toks)
        assert ores["overflow"] == (u <= 3)
        for m in ms:
            assert decisions(m.result(u)) == oracle_decisions(ores), (u, m.rank)
    grp.close()


@pytest.mark.parametrize("world,ce,sharded", [(4, 1, False), (8, 0, False), (3, 0, True)])
def test_virtual_accum_fp32(world, ce, sharded):
    """SURVEY Z1's fp32-accumulator knob at W > 1: per-rank binary32 sums, rn16 of the last one, then the same fp16
    all-reduce (SM or copy engines) and decisions; R bitwise the oracle's binary32 variant (orc_accumulate32)."""
    _run(world, "real", sharded, mode="buckets", acc32=True, ar_copy_engine=ce)


@pytest.mark.parametrize("world,sharded", [(4, False), (7, True)])
def test_virtual_accumulate_many(world, sharded):
    _run(world, "real", sharded, mode="many")


@pytest.mark.parametrize("world,sharded", [(8, False), (6, True)])
def test_virtual_rank_major_order_exact_family(world, sharded):
    """Rank-major calls (rank W-1 first, each rank all its micro-batches) with G_exact."""
    _run(world, "exact", sharded, mode="rank_major")


def test_virtual_world_invariance_w8():
    """(W = 8, c = 1) over 8 virtual ranks == (1, c = 8) on one ctx, bit for bit with G_real (SURVEY c.3): the
    fused all-reduce adds rank by rank exactly as one rank accumulates micro-batch by micro-batch."""
    import paper_1806_00187_b200 as P
    W = 8
    wl8 = models.Workload("inv", TENSORS, W, 1, family="real")
    wl1 = models.Workload("inv", TENSORS, 1, W, family="real")
    lay = synth.Layout(wl8)
    theta0 = synth.theta0_cpu(wl8, lay)
    grp = P.VirtualGroup(wl8.numel, theta0, lib_cfg(wl8, bucket_bytes=400_000), world=W)
    one = P.UpdateStep(wl1.numel, theta0, lib_cfg(wl1, bucket_bytes=400_000, fuse_final=0))
    e = 7
    for u in range(1, 4):
        g = [synth.micro_grad_cpu(wl8, lay, u, r, 1, e) for r in range(W)]
        t = [synth.ntokens(wl8, u, r, 1) for r in range(W)]
        for r in range(W):
            grp.members[r].accumulate(h2t(g[r]), t[r])
        for k in range(W):
            one.accumulate(h2t(g[k]), t[k])
        for m in grp.members:
            m.step(wait=False)
        r1 = one.step()
        assert decisions(grp.members[0].result(u)) == decisions(r1)
        a, b = gpu_state(grp.members[W - 1]), gpu_state(one)
        for k in a:
            assert np.array_equal(a[k], b[k]), (u, k)
        e = r1["scale_log2_next"]
    grp.close()
    one.close()


def test_virtual_group_call_rules():
    """include/smpu.h's two rules for group members, each an ESTATE that leaves the group usable; graphs refused."""
    import paper_1806_00187_b200 as P
    W = 3
    wl = models.Workload("rules", [("w", 40_000, 0)], W, 2, family="real")
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    for sharded in (0, 1):
        grp = P.VirtualGroup(wl.numel, theta0, lib_cfg(wl, sharded=sharded), world=W)
        ms = grp.members
        g = [[h2t(synth.micro_grad_cpu(wl, lay, 1, r, k, 7)) for k in (1, 2)] for r in range(W)]
        for r in range(W):
            ms[r].accumulate(g[r][0], 100)
        ms[0].accumulate(g[0][1], 100)
        with pytest.raises(P.SmpuError) as ei:     # rank 1 and 2 have not given their last micro-batch
            ms[0].step(wait=False)
        assert ei.value.status == P.smpu.ESTATE
        for r in (1, 2):
            ms[r].accumulate(g[r][1], 100)
        if sharded:
            with pytest.raises(P.SmpuError) as ei:  # the sharded update completes with the last rank's step
                ms[0].step(wait=True)
            assert ei.value.status == P.smpu.ESTATE
        ms[0].step(wait=False)
        with pytest.raises(P.SmpuError) as ei:     # rank 0's next update waits for the round to close
            ms[0].accumulate(g[0][0], 100)
        assert ei.value.status == P.smpu.ESTATE
        ms[1].step(wait=False)
        ms[2].step(wait=False)
        res = [m.result(1) for m in ms]
        assert all(x["applied"] == 1 and x["ntokens_total"] == 600 for x in res)
        with pytest.raises(P.SmpuError) as ei:
            ms[1].graph_capture([g[1][0], g[1][1]])
        assert ei.value.status == P.smpu.EINVAL
        ms[0].accumulate(g[0][0], 100)              # the round closed: next update is open
        grp.close()


def test_c3_enfr_first_period_virtual_w8(gold):
    """BASELINE.json configs[3] at its stated world size: Transformer-big En-Fr (221.9M params) over 8 ranks,
    update_freq 16, with the INF / NAN / ACC_OVF / RED_OVF burst at u = 2500-2503 -- here as 8
    virtual ranks on one GPU (28 GB of rank state).  The schedule is periodic (the same burst again at 5000-5003
    after the same regrowth), so this runs its first period, u = 1..2600: the growth at 2000 clean updates, the
    four skips with the scale halved each time, the clean restart.  The whole 5,200 updates run at W = 1
    (test_gpu_fullsize.py) and at W = 4 on real peers (test_gpu_multi.py); here the generator's 128 full-size
    micro-gradients per update are the cost (~0.14 s per update).  Decisions bitwise against the sampled-index
    oracle every update (the bounded G_exact generator cannot overflow alone, so the schedule decides, SURVEY
    8(d.4)), the hand-derived scaler checkpoints, sampled theta/m/v/w16 at the end (1e-4), replicas bitwise
    identical on the device."""
    updates = 2600
    import torch
    import paper_1806_00187_b200 as P
    W = 8
    wl = models.big_enfr(world=W)
    lay = synth.Layout(wl)
    c = wl.update_freq
    theta0 = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    grp = P.VirtualGroup(wl.numel, theta0, lib_cfg(wl), world=W)
    del theta0
    ms = grp.members
    rng = np.random.default_rng(3)
    bb = ms[0].bucket_begin
    idx = np.unique(np.concatenate([rng.integers(0, lay.n, 2048), lay.begin[1:-1], bb[1:-1], bb[1:-1] - 1,
                                    [inj["i"] for inj in wl.injections]])).astype(np.int64)
    orc = O.Oracle(synth.theta0_sample(wl, idx))
    mags = Magnitudes(orc.theta.copy())
    checks = {int(r[0]): tuple(map(int, r[1:])) for r in gold("scaler_trace_c3.txt")}
    inj_u = {inj["u"] for inj in wl.injections}
    # each rank's 16 micro-batches resident, accumulated in one pass (smpu_accumulate_many: the same sums in the same
    # order as 16 calls, bitwise -- tests/test_gpu_parity.py); the buffers are reused rank after rank, stream-ordered
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(c)]
    pending = []
    e = 7
    for u in range(1, updates + 1):
        for r in range(W):
            for k in range(1, c + 1):
                synth.micro_grad_gpu(bufs[k - 1], wl, lay, u, r, k, e)
            ms[r].accumulate_many(bufs, [synth.ntokens(wl, u, r, k) for k in range(1, c + 1)])
        for m in ms:
            m.step(wait=False)
        grads = [[synth.micro_grad_sample(wl, lay, idx, u, r, k, e) for k in range(1, c + 1)] for r in range(W)]
        toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(W)]
        before = snapshot(orc)
        ores = orc.update(grads, toks, overflow=(u in inj_u))
        if ores["applied"]:
            mags.update(ores["R"], ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
        if u in checks:
            assert (orc.e, orc.s.clean, orc.s.t) == checks[u], u
        pending.append((u, oracle_decisions(ores)))
        e = orc.e
        if len(pending) >= 32 or u == updates:
            for uu, od in pending:
                for m in ms:
                    assert decisions(m.result(uu)) == od, (uu, m.rank)
            pending = []
    assert sum(1 for u in checks if u <= updates) == 5
    report = []
    check_state(gpu_state(ms[0], idx), snapshot(orc), mags, 1e-4, where=f"after {updates} updates", report=report)
    s = ms[0].scalars()
    # after 2503: e = 4, clean 0, t = 2499 (golden); 97 clean updates later
    assert (s["e"], s["clean"], s["t"], s["attempts"]) == (4, 97, 2596, 2600) == (orc.e, orc.s.clean, orc.s.t, 2600)
    for which, dt in ((P.smpu.STATE_MASTER, torch.float32), (P.smpu.STATE_M, torch.float32),
                      (P.smpu.STATE_V, torch.float32), (P.smpu.STATE_W16, torch.int16)):
        ref = torch.empty(lay.n, dtype=dt, device="cuda")
        ms[0].get_state(which, out=ref)
        other = torch.empty_like(ref)
        for m in ms[1:]:
            m.get_state(which, out=other)
            assert torch.equal(ref, other), (which, m.rank)
        del ref, other
    grp.close()
    print("C3 virtual W=8:", format_report(report))
