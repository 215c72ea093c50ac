"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (150 MiB buckets, the
library's persistent grids, whole-micro-batch accumulate calls, device-resident GPU-generated inputs).

* configs[1] Transformer-base En-De (60.9M params, c = 1): every element against the full-vector oracle.
* configs[2] Transformer-big En-De (209.9M params, c = 16): sampled outputs (4096 random indices + every
  tensor and bucket boundary and its neighbours + injected indices), each computed one by one by the
  oracle; the overflow decision of the clean update is taken by the oracle over the full vector.
* configs[3] Transformer-big En-Fr (221.9M params, c = 16) with periodic injected overflow: all 5,200
  updates, decisions bitwise every update (hand-derived checkpoints in tests/golden/scaler_trace_c3.txt),
  sampled state parity at the end.  At W = 1 the RED_OVF kind becomes NINF (synth/models.py).
"""
import numpy as np
import pytest

import oracle as O
import synth
from synth import models
from tests.gpu_util import (RTOL_1, RTOL_100, Magnitudes, check_state, decisions, gpu_state, lib_cfg,
                            oracle_decisions, snapshot)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_1806_00187_b200 as pkg
    return pkg


def _sample_idx(lay, bucket_begin, extra=(), n_random=4096, seed=0):
    rng = np.random.default_rng(seed)
    b = np.concatenate([lay.begin, bucket_begin])
    idx = np.concatenate([rng.integers(0, lay.n, n_random), b, b - 1, b + 1, b + 15, b + 16, list(extra)])
    return np.unique(idx[(idx >= 0) & (idx < lay.n)]).astype(np.int64)


def _gpu_inputs(wl, lay, u, r, e, bufs):
    for k in range(1, wl.update_freq + 1):
        synth.micro_grad_gpu(bufs[k - 1], wl, lay, u, r, k, e)


def test_base_ende_full_vector(P):
    import torch
    wl = models.base_ende()
    lay = synth.Layout(wl)
    theta0 = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))                  # default: fused last micro-batch
    ref = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))     # stores R: checked bitwise
    th0 = synth.theta0_cpu(wl, lay)
    assert np.array_equal(theta0.cpu().numpy(), th0)
    orc = O.Oracle(th0)
    mags = Magnitudes(th0)
    buf = [torch.empty(lay.n, dtype=torch.int16, device="cuda")]
    for u in (1, 2, 3):
        e = orc.e
        _gpu_inputs(wl, lay, u, 0, e, buf)
        tok = synth.ntokens(wl, u, 0, 1)
        step.accumulate(buf[0], tok)
        res = step.step()
        ref.accumulate(buf[0], tok)
        rres = ref.step()
        before = snapshot(orc)
        ores = orc.update([[synth.micro_grad_cpu(wl, lay, u, 0, 1, e)]], [[tok]])
        assert decisions(res) == decisions(rres) == oracle_decisions(ores)
        assert np.array_equal(ref.get_state(P.smpu.STATE_ACCUM), ores["R"])
        mags.update(ores["R"], ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
        got = gpu_state(step)
        check_state(got, snapshot(orc), mags, RTOL_1 if u == 1 else 1e-5, where=f"update {u}")
        for name, arr in gpu_state(ref).items():
            assert np.array_equal(got[name], arr), f"update {u}: fused {name} differs from the unfused path"


@pytest.mark.parametrize("final", ["whole", "bucket"])
def test_big_ende_sampled(P, final):
    import torch
    inj = [dict(u=2, kind="INF", r=0, k=9, i=123_456_789)]
    wl = models.big_ende()
    wl.injections = inj
    lay = synth.Layout(wl)
    theta0 = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))   # stores R: checked (sampled) bitwise
    fstep = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))                # the default, fused last micro-batch
    assert step.n_buckets == 3
    idx = _sample_idx(lay, step.bucket_begin, extra=[123_456_789])
    orc = O.Oracle(synth.theta0_sample(wl, idx))
    mags = Magnitudes(orc.theta.copy())
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(wl.update_freq)]
    for u in (1, 2, 3):
        e = orc.e
        _gpu_inputs(wl, lay, u, 0, e, bufs)
        toks = [synth.ntokens(wl, u, 0, k) for k in range(1, wl.update_freq + 1)]
        for st in (step, fstep):
            for k in range(wl.update_freq):
                if final == "bucket" and k == wl.update_freq - 1:
                    st.micro_begin(toks[k])
                    bb = st.bucket_begin
                    for b in (2, 0, 1):
                        st.accumulate_bucket(b, bufs[k][bb[b]:bb[b + 1]])
                else:
                    st.accumulate(bufs[k], toks[k])
        res = step.step()
        assert decisions(fstep.step()) == decisions(res), u
        grads = [[synth.micro_grad_sample(wl, lay, idx, u, 0, k, e) for k in range(1, wl.update_freq + 1)]]
        overflow = O.full_overflow(wl, lay, u, e) if u == 1 else (u == 2)
        before = snapshot(orc)
        ores = orc.update(grads, [toks], overflow=overflow)
        assert decisions(res) == oracle_decisions(ores), (u, res, ores)
        acc = step.get_state(P.smpu.STATE_ACCUM)[idx]
        fin = (ores["R"] & 0x7C00) != 0x7C00
        assert np.array_equal(acc[fin], ores["R"][fin])
        assert np.array_equal(acc[~fin] & 0x7C00, ores["R"][~fin] & 0x7C00)
        if ores["applied"]:
            mags.update(ores["R"], ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
        got = gpu_state(step, idx)
        check_state(got, snapshot(orc), mags, RTOL_1 if u == 1 else 1e-5, where=f"update {u}")
        for name, arr in gpu_state(fstep, idx).items():
            assert np.array_equal(got[name], arr), f"update {u}: fused {name} differs from the unfused path"


def test_big_enfr_5200_updates_periodic_overflow(P, gold):
    import torch
    wl = models.big_enfr(world=1)
    lay = synth.Layout(wl)
    theta0 = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    inj_idx = [inj["i"] for inj in wl.injections]
    idx = _sample_idx(lay, step.bucket_begin, extra=inj_idx, n_random=2048)
    orc = O.Oracle(synth.theta0_sample(wl, idx))
    mags = Magnitudes(orc.theta.copy())
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(wl.update_freq)]
    inj_u = {inj["u"] for inj in wl.injections}
    checks = {int(r[0]): tuple(map(int, r[1:])) for r in gold("scaler_trace_c3.txt")}
    pending = []
    for u in range(1, wl.updates + 1):
        e = orc.e
        _gpu_inputs(wl, lay, u, 0, e, bufs)
        toks = [synth.ntokens(wl, u, 0, k) for k in range(1, wl.update_freq + 1)]
        for k in range(wl.update_freq):
            step.accumulate(bufs[k], toks[k])
        step.step(wait=False)
        # the bounded exact generator cannot overflow by itself: the decision is the schedule's
        grads = [[synth.micro_grad_sample(wl, lay, idx, u, 0, k, e) for k in range(1, wl.update_freq + 1)]]
        before_th = orc.theta.copy()
        ores = orc.update(grads, [toks], overflow=(u in inj_u))
        if ores["applied"]:
            mags.update(ores["R"], ores["e_used"], ores["N"], before_th, orc.theta)
        pending.append((u, oracle_decisions(ores)))
        if u in checks:
            assert (orc.e, orc.s.clean, orc.s.t) == checks[u], u
        if len(pending) >= 32 or u == wl.updates:
            for uu, od in pending:
                assert decisions(step.result(uu)) == od, uu
            pending = []
    check_state(gpu_state(step, idx), snapshot(orc), mags, RTOL_100, where="after 5200 updates")
    s = step.scalars()
    assert (s["e"], s["clean"], s["t"], s["attempts"]) == (1, 197, 5192, 5200)


def test_more_than_2_31_elements(P):
    """Maximum-size edge: a 2^31 + 2^20 + 9 element vector (64-bit indexing in every kernel, 43 GB of HBM),
    odd tensor sizes so the last buckets start unaligned; sampled parity incl. elements beyond 2^31, a skip."""
    import torch
    n_big = (1 << 31) + (1 << 20) + 9
    tensors = [("w0", (1 << 30) + 3, 0), ("b0", 1001, 1), ("w1", n_big - ((1 << 30) + 3) - 1001 - 4097, 0),
               ("e", 4097, 2)]
    inj = [dict(u=2, kind="NINF", r=0, k=2, i=(1 << 31) + 12345)]
    wl = models.Workload("huge", tensors, 1, 2, injections=inj)
    lay = synth.Layout(wl)
    assert lay.n == n_big
    theta0 = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, bucket_bytes=1 << 30))
    del theta0
    torch.cuda.empty_cache()
    idx = _sample_idx(lay, step.bucket_begin, extra=[(1 << 31) - 1, 1 << 31, (1 << 31) + 12345, lay.n - 1],
                      n_random=2048)
    orc = O.Oracle(synth.theta0_sample(wl, idx))
    mags = Magnitudes(orc.theta.copy())
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(2)]
    for u in (1, 2, 3):
        e = orc.e
        _gpu_inputs(wl, lay, u, 0, e, bufs)
        toks = [synth.ntokens(wl, u, 0, k) for k in (1, 2)]
        step.accumulate(bufs[0], toks[0])
        step.accumulate(bufs[1], toks[1])
        res = step.step()
        grads = [[synth.micro_grad_sample(wl, lay, idx, u, 0, k, e) for k in (1, 2)]]
        before = orc.theta.copy()
        ores = orc.update(grads, [toks], overflow=(u == 2))
        assert decisions(res) == oracle_decisions(ores), (u, res, ores)
        if ores["applied"]:
            mags.update(ores["R"], ores["e_used"], ores["N"], before, orc.theta)
        sel = torch.from_numpy(idx).cuda()
        gpu = {}
        for name, which in (("theta", P.smpu.STATE_MASTER), ("m", P.smpu.STATE_M), ("v", P.smpu.STATE_V),
                            ("w16", P.smpu.STATE_W16)):
            full = step.get_state(which)
            gpu[name] = full[idx]
            del full
        check_state(gpu, snapshot(orc), mags, RTOL_1 if u == 1 else 1e-5, where=f"update {u}")
        del sel
