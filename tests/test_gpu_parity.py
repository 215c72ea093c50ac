"""CUDA path (libsmpu.so through its C ABI) vs the CPU oracle, element by element on the same seeded inputs.

Bar (north_star): decisions (overflow, applied, e_used, e_next, lr bits, t, N, clean) bitwise
every update; accumulator bitwise at W = 1; w16 within 1 fp16 ulp; theta/m/v within 1e-6 (operand-scale
relative) after 1 update and 1e-4 after 100.

At W = 1 the library's default fuses the last micro-batch into Adam (fuse_final: R is never stored), so the
runner drives two ctxs with the same inputs: fuse_final = 0, whose accumulator is checked bitwise against the
oracle's R and whose state against the oracle, and the default one, which must agree with it bit for bit
(decisions, theta/m/v, w16) every update.
"""
import numpy as np
import pytest

import oracle as O
import synth
from synth import models
from tests.gpu_util import (RTOL_1, RTOL_100, Magnitudes, check_state, decisions, format_report, gpu_state, h2t,
                            lib_cfg, oracle_decisions, rtol_for, snapshot)

pytestmark = pytest.mark.gpu
REPORT = []   # worst err/D of every W = 1 runner (printed by test_zz_error_report)


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_1806_00187_b200 as pkg
    return pkg


def run_pair(P, wl, updates, *, ocfg=None, cfg_kw=None, mode="whole", rtol_last=None, check_every=True,
             host_inputs=None, bucket_order=None):
    """Run the library and the oracle (full vectors) side by side; compare after every update."""
    import torch
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    ocfg = ocfg or O.Config()
    orc = O.Oracle(theta0, ocfg)
    kw = dict(cfg_kw or {})
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, ocfg, **dict(kw, fuse_final=0)))
    fstep = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, ocfg, **kw)) if wl.world == 1 else None
    assert step.n == lay.n
    mags = Magnitudes(theta0)
    applied = 0
    for u in range(1, updates + 1):
        e = orc.e
        grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, e) for k in range(1, wl.update_freq + 1)]
                 for r in range(wl.world)]
        toks = [[synth.ntokens(wl, u, r, k) for k in range(1, wl.update_freq + 1)] for r in range(wl.world)]
        before = snapshot(orc)
        ores = orc.update(grads, toks)
        for k in range(wl.update_freq):
            g = grads[0][k]
            if host_inputs == "pageable":
                src = g
            elif host_inputs == "pinned":
                src = torch.from_numpy(g.view(np.int16)).pin_memory()
            else:
                src = h2t(g)
            for st in (step, fstep) if fstep is not None else (step,):
                if mode == "whole":
                    st.accumulate(src, toks[0][k])
                else:
                    st.micro_begin(toks[0][k])
                    order = bucket_order(st.n_buckets) if bucket_order else range(st.n_buckets)
                    bb = st.bucket_begin
                    for b in order:
                        st.accumulate_bucket(b, src[bb[b]:bb[b + 1]])
        res = step.step()
        assert decisions(res) == oracle_decisions(ores), f"update {u}: {res} vs {ores}"
        if fstep is not None:
            fres = fstep.step()
            assert decisions(fres) == decisions(res), f"update {u}: fused {fres} vs {res}"
            a_, b_ = gpu_state(fstep), gpu_state(step)
            for name in ("theta", "m", "v", "w16"):
                assert np.array_equal(a_[name], b_[name]), f"update {u}: fused {name} differs"
        acc = step.get_state(P.smpu.STATE_ACCUM)
        R = ores["R"]
        nan = np.isnan(R.view(np.float16))
        assert np.array_equal(np.isnan(acc.view(np.float16)), nan)
        assert np.array_equal(acc[~nan], R[~nan]), f"update {u}: accumulator differs"
        if ores["applied"]:
            applied += 1
            mags.update(R, ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
        if check_every or u == updates:
            rtol = rtol_for(applied) if rtol_last is None else min(rtol_for(applied), rtol_last)
            check_state(gpu_state(step), snapshot(orc), mags, rtol, where=f"update {u}", report=REPORT)
    return step, orc


def test_tiny_config_ten_updates_with_injected_inf(P):
    """BASELINE configs[0]: 1M params, world=1, update_freq=2, 10 updates, +inf at (u=5, r=0, k=2, i=123457)."""
    run_pair(P, models.tiny(), 10, rtol_last=1e-5)


def test_tiny_hundred_updates(P):
    wl = models.tiny(updates=100, injections=[dict(u=37, kind="NAN", r=0, k=1, i=5)])
    run_pair(P, wl, 100, check_every=False)


def test_first_update_within_1e6(P):
    run_pair(P, models.tiny(injections=[]), 1)


@pytest.mark.parametrize("kind", ["INF", "NINF", "NAN", "ACC_OVF"])
def test_injection_kinds_skip_bitwise(P, kind):
    inj = [dict(u=2, kind=kind, r=0, k=2, i=999_983)]
    wl = models.Workload("inj", [("w", 1_000_000, 0)], 1, 3, injections=inj)
    run_pair(P, wl, 3)


def test_ragged_tensors_small_buckets_bucket_mode_out_of_order(P):
    # odd sizes -> bucket starts not 16-aligned; tiny buckets; 3 micro-batches; buckets given in reverse order
    tensors = [("a", 1, 0), ("b", 17, 1), ("c", 100_003, 0), ("d", 5, 1), ("e", 65_536, 2), ("f", 33, 1),
               ("g", 250_001, 0)]
    wl = models.Workload("ragged", tensors, 1, 3, injections=[dict(u=3, kind="INF", r=0, k=3, i=100_020)])
    step, _ = run_pair(P, wl, 5, cfg_kw=dict(bucket_bytes=64 * 1024), mode="bucket",
                       bucket_order=lambda nb: list(reversed(range(nb))), rtol_last=1e-5)
    assert step.n_buckets == 3 and step.bucket_begin[1] % 16 != 0


@pytest.mark.parametrize("host", ["pinned", "pageable"])
def test_host_buffers(P, host):
    wl = models.Workload("host", [("w", 40_000_001, 0), ("b", 7, 1)], 1, 2)  # > one 32 MiB staging chunk
    run_pair(P, wl, 2, host_inputs=host)


def test_growth_and_clamps(P):
    # growth after 3 clean updates, max 2^9; an overflow at u=8; min clamp at 2^6
    ocfg = O.Config(growth=3, init_scale_log2=7, max_scale_log2=9, min_scale_log2=6)
    inj = [dict(u=8, kind="INF", r=0, k=1, i=3), dict(u=9, kind="INF", r=0, k=2, i=4),
           dict(u=10, kind="NAN", r=0, k=1, i=5)]
    wl = models.Workload("grow", [("w", 4096, 0), ("b", 64, 1)], 1, 2, injections=inj)
    run_pair(P, wl, 16, ocfg=ocfg, rtol_last=1e-5)


def test_two_x_lr_and_update_freq_1(P):
    ocfg = O.Config(peak_lr=1e-3)   # "2x lr"
    wl = models.Workload("c1", [("w", 300_000, 0), ("e", 70_000, 2)], 1, 1)
    run_pair(P, wl, 4, ocfg=ocfg, rtol_last=1e-5)


@pytest.mark.parametrize("mode,host", [("whole", None), ("bucket", None), ("whole", "pinned")])
def test_accum_fp32_knob(P, mode, host):
    """SURVEY Z1 knob (smpu_config.accum_fp32): fp32 sums, rn16 of the last one, against the oracle's binary32
    variant -- the reduced gradient bitwise, decisions bitwise, state within tolerance -- through an overflow that
    only the fp16 accumulator would raise, one that both raise, and a NaN."""
    tensors = [("a", 17, 1), ("b", 100_003, 0), ("c", 65_536, 2), ("d", 9, 1)]
    inj = [dict(u=2, kind="ACC_OVF", r=0, i=70_000), dict(u=4, kind="NAN", r=0, k=2, i=100_019),
           dict(u=5, kind="INF", r=0, k=1, i=3)]
    wl = models.Workload("acc32", tensors, 1, 4, injections=inj)
    run_pair(P, wl, 6, ocfg=O.Config(accum_fp32=True), cfg_kw=dict(bucket_bytes=64 * 1024), mode=mode,
             host_inputs=host, rtol_last=1e-5)


def test_accum_fp32_many_and_inplace(P):
    """accum_fp32 through accumulate_many (one pass per micro-batch) and an in-place producer adding into the fp32
    accumulator (torch fp32 adds are binary32 round-to-nearest): bitwise the streaming fp32 path."""
    import torch
    tensors = [("a", 17, 1), ("b", 100_003, 0), ("c", 65_536, 2)]
    wl = models.Workload("acc32m", tensors, 1, 5, injections=[dict(u=3, kind="NAN", r=0, k=4, i=100_010)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    ocfg = O.Config(accum_fp32=True)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, ocfg))
    b = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, ocfg))
    x = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, ocfg, bucket_bytes=100_000))
    acc = torch.as_tensor(_DevView(x.accumulator_ptr(), lay.n, "<f4"), device="cuda")
    orc = O.Oracle(theta0, ocfg)
    for u in range(1, 5):
        e = orc.e
        grads = [synth.micro_grad_cpu(wl, lay, u, 0, k, e) for k in range(1, 6)]
        toks = [synth.ntokens(wl, u, 0, k) for k in range(1, 6)]
        ores = orc.update([grads], [toks])
        dev = [h2t(g) for g in grads]
        for k in range(5):
            a.accumulate(dev[k], toks[k])
        b.accumulate_many(dev[:3], toks[:3])
        b.accumulate_many(dev[3:], toks[3:])
        for k in range(5):
            g32 = dev[k].view(torch.float16).float()
            acc.copy_(g32) if k == 0 else acc.add_(g32)
            if k < 4:
                x.accumulate(None, toks[k])
            else:
                x.micro_begin(toks[k])
                for bk in reversed(range(x.n_buckets)):
                    x.accumulate_bucket(bk, None)
        ra, rb, rx = a.step(), b.step(), x.step()
        assert decisions(ra) == decisions(rb) == decisions(rx) == oracle_decisions(ores), u
        R = ores["R"]
        nan = np.isnan(R.view(np.float16))
        for st in (a, b, x):
            got = st.get_state(P.smpu.STATE_ACCUM)
            assert np.array_equal(np.isnan(got.view(np.float16)), nan) and np.array_equal(got[~nan], R[~nan]), u
        for w in (0, 1, 2, 3, 5):
            sa = a.get_state(w)
            assert np.array_equal(sa, b.get_state(w)) and np.array_equal(sa, x.get_state(w)), (u, w)


def test_split_tensor_buckets(P):
    """smpu_config.split_tensors: fixed 128-element-aligned buckets cut through tensors.  Whole, bucket-wise (random
    order) and in-place per-tensor-hook micro-batches give the default plan's bits (buckets change timing, never
    values); a tensor spanning several buckets is counted in each by smpu_tensor_ready."""
    import torch
    tensors = [("a", 17, 1), ("b", 300_001, 0), ("c", 65_536, 2), ("d", 9, 1)]
    wl = models.Workload("split", tensors, 1, 3, injections=[dict(u=2, kind="NAN", r=0, k=3, i=150_000)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    x = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, bucket_bytes=100_000, split_tensors=1))
    per = 50_048
    assert x.bucket_begin.tolist() == list(range(0, lay.n, per)) + [lay.n]
    acc = torch.as_tensor(_DevView(x.accumulator_ptr(), lay.n), device="cuda")
    orc = O.Oracle(theta0)
    rng = np.random.default_rng(5)
    for u in range(1, 5):
        e = orc.e
        grads = [synth.micro_grad_cpu(wl, lay, u, 0, k, e) for k in (1, 2, 3)]
        toks = [synth.ntokens(wl, u, 0, k) for k in (1, 2, 3)]
        ores = orc.update([grads], [toks])
        dev = [h2t(g) for g in grads]
        for k in range(3):
            a.accumulate(dev[k], toks[k])
        x.accumulate(dev[0], toks[0])
        x.micro_begin(toks[1])
        bb = x.bucket_begin
        for b in rng.permutation(x.n_buckets):
            x.accumulate_bucket(int(b), dev[1][bb[b]:bb[b + 1]])
        acc.add_(dev[2].view(torch.float16))            # the in-place producer's last micro-batch
        x.micro_begin(toks[2])
        for j in rng.permutation(len(tensors)):
            x.tensor_ready(int(j))
        ra, rx = a.step(), x.step()
        assert decisions(ra) == decisions(rx) == oracle_decisions(ores), u
        for w in (0, 1, 2, 3, 5):
            assert np.array_equal(a.get_state(w), x.get_state(w)), (u, w)


def test_bucket_size_invariance(P):
    # buckets change timing, never values: final state bitwise equal for any bucket size
    import torch
    wl = models.Workload("binv", [(f"t{j}", 50_000 + 1000 * j, j % 2) for j in range(12)], 1, 2)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    finals = []
    for bb in (2 * 60_000, 1 << 20, 150 << 20):
        step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, bucket_bytes=bb))
        e = 7
        for u in range(1, 4):
            for k in (1, 2):
                g = h2t(synth.micro_grad_cpu(wl, lay, u, 0, k, e))
                step.micro_begin(3000)
                for b in range(step.n_buckets):
                    step.accumulate_bucket(b, g[step.bucket_begin[b]:step.bucket_begin[b + 1]])
            e = step.step()["scale_log2_next"]
        finals.append([step.get_state(w).copy() for w in range(5)])
        torch.cuda.synchronize()
    for other in finals[1:]:
        for a, b in zip(finals[0], other):
            assert np.array_equal(a, b)


def test_resume_bitwise(P):
    wl = models.tiny(injections=[dict(u=4, kind="INF", r=0, k=1, i=11)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)

    def drive(step, us):
        for u in us:
            e = int(step.scalars()["e"])
            for k in (1, 2):
                step.accumulate(h2t(synth.micro_grad_cpu(wl, lay, u, 0, k, e)), synth.ntokens(wl, u, 0, k))
            step.step()

    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    drive(a, range(1, 7))
    b = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    drive(b, range(1, 4))
    saved = [b.get_state(w).copy() for w in (0, 1, 2, 3, 5)]
    c = P.UpdateStep(wl.numel, np.zeros(lay.n, np.float32), lib_cfg(wl))
    for w, arr in zip((0, 1, 2, 3, 5), saved):
        c.set_state(w, arr)
    drive(c, range(4, 7))
    for w in (0, 1, 2, 3, 5):
        assert np.array_equal(a.get_state(w), c.get_state(w)), w


def test_async_step_and_result_ring(P):
    wl = models.Workload("async", [("w", 200_000, 0)], 1, 1)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    orc = O.Oracle(theta0)
    ores = []
    for u in range(1, 6):
        g = synth.micro_grad_cpu(wl, lay, u, 0, 1, 7)
        step.accumulate(h2t(g), 1000 + u)
        step.step(wait=False)
        ores.append(orc.update([[g]], [[1000 + u]]))
    for u in range(1, 6):
        assert decisions(step.result(u)) == oracle_decisions(ores[u - 1])
    with pytest.raises(P.SmpuError):
        step.result(99)


def test_call_order_errors_and_discard(P):
    import torch
    wl = models.Workload("err", [("w", 1000, 0)], 1, 2)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    g = h2t(synth.micro_grad_cpu(wl, lay, 1, 0, 1, 7))
    with pytest.raises(P.SmpuError) as ei:
        step.step()                                    # no micro-batch yet
    assert ei.value.status == P.smpu.ESTATE
    step.accumulate(g, 0)
    with pytest.raises(P.SmpuError):
        step.accumulate_bucket(0, g)                   # no micro_begin
    step.accumulate(g, 0)
    with pytest.raises(P.SmpuError):
        step.accumulate(g, 5)                          # third micro-batch with c = 2
    before = [step.get_state(w).copy() for w in (0, 1, 2, 3, 5)]
    with pytest.raises(P.SmpuError) as ei:
        step.step()                                    # N = 0: discarded (reading R19)
    assert ei.value.status == P.smpu.ESTATE
    after = [step.get_state(w) for w in (0, 1, 2, 3, 5)]
    for a, b in zip(before[:4], after[:4]):
        assert np.array_equal(a, b)
    assert after[4][:3].tolist() == before[4][:3].tolist()   # e, clean, t unchanged
    with pytest.raises(P.SmpuError) as ei:
        step.micro_begin(-1)
    assert ei.value.status == P.smpu.EINVAL
    torch.cuda.synchronize()


class _DevF32:
    """A device fp32 scalar owned by the library, viewed (not copied) through __cuda_array_interface__."""

    def __init__(self, ptr):
        self.__cuda_array_interface__ = {"shape": (1,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def test_loss_scale_pointer_tracks_scaler(P):
    import torch
    wl = models.Workload("ls", [("w", 4096, 0)], 1, 1, injections=[dict(u=2, kind="INF", r=0, k=1, i=0)])
    lay = synth.Layout(wl)
    step = P.UpdateStep(wl.numel, synth.theta0_cpu(wl, lay), lib_cfg(wl))
    scale = torch.as_tensor(_DevF32(step.loss_scale_ptr()), device="cuda")
    assert scale.item() == 2.0 ** 7
    for u in (1, 2):
        step.accumulate(h2t(synth.micro_grad_cpu(wl, lay, u, 0, 1, 7)), 100)
        res = step.step()
        assert scale.item() == 2.0 ** res["scale_log2_next"]
    assert res["overflow"] == 1 and scale.item() == 2.0 ** 6


def test_graph_replay_bitwise_equals_call_path(P):
    """smpu_graph_capture / smpu_graph_launch: the same update as c x accumulate + step, bit for bit, with the
    token counts read at replay time and the decisions the oracle's (injected overflow at u = 3)."""
    import torch
    wl = models.Workload("graph", [("w", 300_001, 0), ("e", 65_536, 2), ("b", 33, 1)], 1, 3,
                         injections=[dict(u=3, kind="INF", r=0, k=2, i=77)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    b = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    orc = O.Oracle(theta0)
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(3)]
    a.kernel_stats(reset=True)
    b.kernel_stats(reset=True)      # drops init's theta -> w16 cast
    b.graph_capture(bufs)
    assert sum(v["launches"] for v in b.kernel_stats(reset=True).values()) == 0   # capturing launches nothing
    for u in range(1, 7):
        e = orc.e
        grads = [synth.micro_grad_cpu(wl, lay, u, 0, k, e) for k in (1, 2, 3)]
        toks = [synth.ntokens(wl, u, 0, k) for k in (1, 2, 3)]
        ores = orc.update([grads], [toks])
        for k in range(3):
            a.accumulate(h2t(grads[k]), toks[k])
            bufs[k].copy_(torch.from_numpy(grads[k].view(np.int16)))
        ra = a.step()
        b.graph_launch(toks)
        rb = b.result(u)
        assert decisions(ra) == decisions(rb) == oracle_decisions(ores), u
        for w in (0, 1, 2, 3, 4, 5):
            assert np.array_equal(a.get_state(w), b.get_state(w)), (u, w)
    # the launch counters (bench.py's gpu_launches) count each replay's kernels like the call path's
    la = {k: v["launches"] for k, v in a.kernel_stats().items()}
    lb = {k: v["launches"] for k, v in b.kernel_stats().items()}
    # fused last micro-batch: first + add + k12 per update; k0 = prep + decide; kc_cast = the (no-op) restore
    assert (la["k1_first"], la["k1_add"], la["k12_fused"], la["k0_decide"], la["kc_cast"], la["k2_adam"]) == \
        (6, 6, 6, 12, 6, 0), la
    assert la == lb, (la, lb)


def test_accumulate_many_bitwise_equals_streaming(P):
    """smpu_accumulate_many (resident micro-batches, one pass) == consecutive smpu_accumulate calls, bit for bit,
    on ragged tensors, mixed with single calls, and as a resident CUDA graph; decisions are the oracle's."""
    import torch
    tensors = [("a", 17, 1), ("b", 100_003, 0), ("c", 65_536, 2), ("d", 5, 1), ("e", 250_001, 0)]
    wl = models.Workload("many", tensors, 1, 5, injections=[dict(u=2, kind="NAN", r=0, k=4, i=100_010),
                                                            dict(u=4, kind="ACC_OVF", r=0, i=77)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    b = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    g = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    orc = O.Oracle(theta0)
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(5)]
    g.graph_capture(bufs, resident=True)
    for u in range(1, 6):
        e = orc.e
        grads = [synth.micro_grad_cpu(wl, lay, u, 0, k, e) for k in range(1, 6)]
        toks = [synth.ntokens(wl, u, 0, k) for k in range(1, 6)]
        ores = orc.update([grads], [toks])
        dev = [h2t(x) for x in grads]
        for k in range(5):
            a.accumulate(dev[k], toks[k])
            bufs[k].copy_(dev[k])
        ra = a.step()
        b.accumulate_many(dev[:2], toks[:2])          # groups of 2, 1, 2
        b.accumulate(dev[2], toks[2])
        b.accumulate_many(dev[3:], toks[3:])
        rb = b.step()
        g.graph_launch(toks)
        rg = g.result(u)
        assert decisions(ra) == decisions(rb) == decisions(rg) == oracle_decisions(ores), u
        # (the accumulator is not compared: the fused last micro-batch consumes R without storing it, so it
        # holds whatever partial sum each grouping stored last)
        for w in (0, 1, 2, 3, 5):
            sa = a.get_state(w)
            assert np.array_equal(sa, b.get_state(w)) and np.array_equal(sa, g.get_state(w)), (u, w)
    with pytest.raises(P.SmpuError) as ei:
        b.accumulate_many(dev + [dev[0]], toks + [1])     # 6 micro-batches with update_freq 5
    assert ei.value.status == P.smpu.ESTATE


class _DevView:
    """A library-owned device array viewed (not copied) by torch through __cuda_array_interface__."""

    def __init__(self, ptr, n, typestr="<f2"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def test_external_accumulation_bitwise(P):
    """SURVEY f3 contract: the producer adds its micro-gradients into smpu_accumulator in place (here torch fp16
    copy/add: rn16(fp32(a)+fp32(b)) == rn16(a+b), innocuous double rounding) and declares them with
    micro_grads=None; the update equals the library-accumulated one bit for bit, decisions the oracle's."""
    import torch
    tensors = [("a", 17, 1), ("b", 100_003, 0), ("c", 65_536, 2)]
    wl = models.Workload("ext", tensors, 1, 3, injections=[dict(u=2, kind="NAN", r=0, k=2, i=50)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    x = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, bucket_bytes=100_000))
    acc = torch.as_tensor(_DevView(x.accumulator_ptr(), lay.n), device="cuda")
    orc = O.Oracle(theta0)
    for u in range(1, 5):
        e = orc.e
        grads = [synth.micro_grad_cpu(wl, lay, u, 0, k, e) for k in (1, 2, 3)]
        toks = [synth.ntokens(wl, u, 0, k) for k in (1, 2, 3)]
        ores = orc.update([grads], [toks])
        for k in range(3):
            g = h2t(grads[k]).view(torch.float16)
            a.accumulate(g.view(torch.int16), toks[k])
            if k == 0:
                acc.copy_(g)
            else:
                acc.add_(g)
            if k < 2:
                x.accumulate(None, toks[k])
            else:                                   # the last one bucket by bucket, as a backward would
                x.micro_begin(toks[k])
                for b in reversed(range(x.n_buckets)):
                    x.accumulate_bucket(b, None)
        ra, rx = a.step(), x.step()
        assert decisions(ra) == decisions(rx) == oracle_decisions(ores), u
        for w in (0, 1, 2, 3, 5):      # accumulators differ by design: x's producer wrote R, a's holds A_2
            assert np.array_equal(a.get_state(w), x.get_state(w)), (u, w)


def test_external_gemm_epilogue_accumulation(P):
    """The f3 producer: dW = dY^T X by cuBLAS with beta = 1 straight into the accumulator.  Measured on B200,
    cuBLAS's fp16 epilogue computes rn16(rn16(alpha * dW_fp32) + A), i.e. the paper's two roundings (reading R1):
    the in-place update is bitwise the same as the GEMM into a scratch buffer followed by the library's K1
    (a second ctx), and both finish identically."""
    import torch
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False   # fp32 accumulation in cuBLAS
    out_f, in_f, T = 384, 256, 3000
    wl = models.Workload("gemm", [("w", out_f * in_f, 0)], 1, 4)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    # fuse_final = 0: the accumulator of the last micro-batch is compared too (the fused path never stores R)
    x = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))
    y = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))
    acc = torch.as_tensor(_DevView(x.accumulator_ptr(), lay.n), device="cuda").view(out_f, in_f)
    scratch = torch.empty(out_f, in_f, dtype=torch.float16, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(0)
    for u in range(1, 3):
        for k in range(4):
            dy = (torch.randn(T, out_f, device="cuda", generator=gen) * 0.05).half()
            xx = (torch.randn(T, in_f, device="cuda", generator=gen) * 0.05).half()
            # in place: beta = 0 for the first micro-batch of the update, 1 after; alpha = the loss scale 2^7
            torch.addmm(acc, dy.t(), xx, beta=0.0 if k == 0 else 1.0, alpha=2.0**7, out=acc)
            x.accumulate(None, T)
            torch.addmm(scratch, dy.t(), xx, beta=0.0, alpha=2.0**7, out=scratch)
            y.accumulate(scratch.view(-1).view(torch.int16), T)
            torch.cuda.synchronize()
            assert np.array_equal(x.get_state(P.smpu.STATE_ACCUM), y.get_state(P.smpu.STATE_ACCUM)), (u, k)
        rx, ry = x.step(), y.step()
        assert decisions(rx) == decisions(ry) and rx["applied"] == 1 and rx["ntokens_total"] == 4 * T
        for w in (0, 1, 2, 3):
            assert np.array_equal(x.get_state(w), y.get_state(w)), (u, w)


def test_graph_direct_c1_bitwise(P):
    """update_freq = 1, W = 1 graph with fuse_final = 0: overflow test in place + Adam reading the producer's
    buffer (no copy) == the (fused, default) call path bit for bit on theta/m/v/w16 and the decisions, through an
    injected NaN."""
    import torch
    wl = models.Workload("direct", [("w", 200_003, 0), ("b", 9, 1)], 1, 1,
                         injections=[dict(u=3, kind="NAN", r=0, k=1, i=200_005)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    g = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))
    orc = O.Oracle(theta0)
    buf = torch.empty(lay.n, dtype=torch.int16, device="cuda")
    g.graph_capture([buf])
    for u in range(1, 6):
        x = synth.micro_grad_cpu(wl, lay, u, 0, 1, orc.e)
        tok = synth.ntokens(wl, u, 0, 1)
        ores = orc.update([[x]], [[tok]])
        a.accumulate(h2t(x), tok)
        ra = a.step()
        buf.copy_(h2t(x))
        g.graph_launch([tok])
        rg = g.result(u)
        assert decisions(ra) == decisions(rg) == oracle_decisions(ores), u
        for w in (0, 1, 2, 3, 5):
            assert np.array_equal(a.get_state(w), g.get_state(w)), (u, w)


def test_graph_direct_c1_misaligned_buffer(P):
    """the c = 1 direct graph path reads the producer's buffer with 256-bit loads, so a buffer that is not
    32-byte aligned (a view at an odd element offset) must take the accumulate path instead -- same bits, no fault."""
    import torch
    wl = models.Workload("direct_mis", [("w", 100_003, 0)], 1, 1)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))
    g = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, fuse_final=0))
    big = torch.empty(lay.n + 1, dtype=torch.int16, device="cuda")
    buf = big[1:]                                   # 2-byte aligned only
    assert buf.data_ptr() % 32 != 0
    g.graph_capture([buf])
    for u in range(1, 4):
        x = synth.micro_grad_cpu(wl, lay, u, 0, 1, 7)
        tok = synth.ntokens(wl, u, 0, 1)
        a.accumulate(h2t(x), tok)
        ra = a.step()
        buf.copy_(h2t(x))
        g.graph_launch([tok])
        assert decisions(g.result(u)) == decisions(ra), u
        for w in (0, 1, 2, 3):
            assert np.array_equal(a.get_state(w), g.get_state(w)), (u, w)


def test_result_of_restored_attempt_is_einval(P):
    """after set_state(SCALARS) the result ring holds none of the restored attempts: smpu_result for
    them is EINVAL instead of a stale record; attempts run after the restore are served."""
    import torch
    wl = models.Workload("ring", [("w", 10_000, 0)], 1, 1)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    st = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    g = torch.zeros(lay.n, dtype=torch.int16, device="cuda")
    st.set_state(P.smpu.STATE_SCALARS, np.array([7, 3, 40, 50], dtype=np.int64))
    for attempt in (1, 50):
        with pytest.raises(P.SmpuError) as ei:
            st.result(attempt)
        assert ei.value.status == P.smpu.EINVAL
    st.accumulate(g, 100)
    st.step(wait=False)
    r = st.result(51)
    assert r["attempt"] == 51 and r["num_updates"] == 41 and r["applied"] == 1
    st.close()


def test_real_training_loop_example(P):
    """examples/train_tiny.py: a real fp16 model whose weights are views of the library's w16, loss scaled by the
    library's device scale, update by libsmpu -- the loss must fall from ln V towards the 10%-noise floor."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "train_tiny", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples",
                                   "train_tiny.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    losses, scales = mod.run(updates=120, verbose=False)
    assert losses[0] > 3.5                      # ~ ln 64 = 4.16 at init
    assert np.mean(losses[-10:]) < 1.5         # learned (noise floor ~0.1*ln 64 + entropy terms)
    assert all(-5 <= s <= 24 for s in scales)


def test_tensor_ready_hooks(P):
    """Per-tensor ready hooks: an in-place producer finishing tensors in a random order; buckets are
    handed over as their last tensor arrives; same bits as the library-accumulated path; misuse is ESTATE."""
    import torch
    tensors = [(f"t{j}", 5_000 + 997 * j, j % 3) for j in range(9)]
    wl = models.Workload("hooks", tensors, 1, 2)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    a = P.UpdateStep(wl.numel, theta0, lib_cfg(wl))
    x = P.UpdateStep(wl.numel, theta0, lib_cfg(wl, bucket_bytes=20_000))
    assert x.n_buckets > 2
    acc = torch.as_tensor(_DevView(x.accumulator_ptr(), lay.n), device="cuda")
    rng = np.random.default_rng(7)
    for u in range(1, 4):
        grads = [h2t(synth.micro_grad_cpu(wl, lay, u, 0, k, 7)).view(torch.float16) for k in (1, 2)]
        toks = [1000 + u, 2000 + u]
        for k in range(2):
            a.accumulate(grads[k].view(torch.int16), toks[k])
            x.micro_begin(toks[k])
            for j in rng.permutation(len(tensors)):
                lo, hi = lay.begin[j], lay.begin[j + 1]
                acc[lo:hi].copy_(grads[k][lo:hi]) if k == 0 else acc[lo:hi].add_(grads[k][lo:hi])
                x.tensor_ready(int(j))
        ra, rx = a.step(), x.step()
        assert decisions(ra) == decisions(rx)
        for w in (0, 1, 2, 3):      # (accumulators differ by design, see test_external_accumulation_bitwise)
            assert np.array_equal(a.get_state(w), x.get_state(w)), (u, w)
    x.micro_begin(10)
    x.tensor_ready(0)
    with pytest.raises(P.SmpuError) as ei:
        x.tensor_ready(0)
    assert ei.value.status == P.smpu.ESTATE


def test_zz_error_report():
    """The W = 1 runners' worst errors under R26's cumulative D (asserted) and SURVEY c.4's one-step D (reported)."""
    if not REPORT:
        pytest.skip("no runner ran")
    print("W = 1 worst errors:", format_report(REPORT))
