"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Every check here compares the oracle with something other than itself: values
printed in PAPER.md / SPEC.md (tests/golden/, cited), closed forms, an
independent library routine (numpy's binary16 converter and arithmetic,
torch._amp_update_scale_, torch.optim.Adam), or brute force on tiny inputs.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synth
from synth import models


def _f(s):
    return float(s)


# ============================================================================ binary16 codec
def test_codec_golden(gold):
    for row in gold("codec_examples.txt"):
        kind, a, b = row[0], row[1], row[2]
        if kind == "d2h":
            assert O.d2h(_f(a)) == int(b, 16), row
        else:
            v = O.h2d(int(a, 16))
            exp = _f(b)
            assert v == exp and math.copysign(1, v) == math.copysign(1, exp), row


def test_codec_exhaustive_round_trip_and_numpy_widening():
    bits = np.arange(65536, dtype=np.uint16)
    x = O.h2d_array(bits)
    ref = bits.view(np.float16).astype(np.float64)           # independent converter (numpy)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(x), nan)
    assert np.array_equal(x[~nan], ref[~nan])
    assert np.array_equal(np.signbit(x[~nan]), np.signbit(ref[~nan]))   # signed zeros
    back = O.d2h_array(x)
    assert np.array_equal(back[~nan], bits[~nan])               # exact round trip
    assert np.all(back[nan] == 0x7E00)                          # canonical NaN


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_codec_rounding_matches_numpy(dtype):
    rng = np.random.default_rng(1)
    n = 1_000_000
    # log-uniform magnitudes spanning underflow .. overflow, random signs, plus exact ties
    mag = np.exp2(rng.uniform(-27, 17, n))
    x = (mag * rng.choice([-1.0, 1.0], n)).astype(dtype)
    h = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    ties = ((h[:-1] + h[1:]) / 2).astype(dtype)                 # every midpoint between neighbours
    x = np.concatenate([x, ties, -ties])
    mine = O.d2h_array(x.astype(np.float64))
    ref = x.astype(np.float16).view(np.uint16)                  # numpy: correctly rounded, RNE
    assert np.array_equal(mine, ref)


# ============================================================================ fp16 addition
def test_hadd_golden(gold):
    for a, b, c, *_ in gold("hadd_examples.txt"):
        r = O.hadd(int(a, 16), int(b, 16))
        if int(c, 16) == 0x7E00:
            assert (r & 0x7C00) == 0x7C00 and (r & 0x3FF)
        else:
            assert r == int(c, 16), (a, b, hex(r))


def test_hadd_matches_numpy_binary16_add():
    # numpy adds binary16 through fp32 (24 >= 2*11+2 bits: innocuous double rounding), an independent
    # implementation of the correctly rounded sum.
    rng = np.random.default_rng(2)
    a = rng.integers(0, 65536, 400_000, dtype=np.uint32).astype(np.uint16)
    b = rng.integers(0, 65536, 400_000, dtype=np.uint32).astype(np.uint16)
    fin = ((a & 0x7C00) != 0x7C00) & ((b & 0x7C00) != 0x7C00)
    a, b = a[fin], b[fin]
    with np.errstate(over="ignore"):
        ref = (a.view(np.float16) + b.view(np.float16)).view(np.uint16)
    acc = a.copy()
    O.lib().orc_accumulate(O._p(acc), O._p(np.ascontiguousarray(b)), acc.size, 0)
    assert np.array_equal(acc, ref)


def test_accumulate_and_reduce_brute_force():
    rng = np.random.default_rng(3)
    W, c, n = 3, 4, 5000
    g = rng.normal(0, 300, (W, c, n)).astype(np.float16)
    accs = []
    for r in range(W):
        a = g[r, 0].copy()                       # first micro-batch: copy (reading R2)
        for k in range(1, c):
            a = (a + g[r, k]).astype(np.float16)
        accs.append(a)
        assert np.array_equal(O.accumulate([g[r, k].view(np.uint16) for k in range(c)]), a.view(np.uint16))
    ref = accs[0].copy()
    for r in range(1, W):                        # ascending rank
        ref = (ref + accs[r]).astype(np.float16)
    assert np.array_equal(O.reduce([a.view(np.uint16) for a in accs]), ref.view(np.uint16))


def test_accumulate_fp32_variant_against_numpy_float32():
    """SURVEY Z1 knob: A32 = fp32(g_1), A32 = fl32(A32 + g_k), then rn16.  Pinned to numpy's IEEE binary32 adds
    and its float32 -> float16 conversion (round to nearest even), including non-finite inputs."""
    rng = np.random.default_rng(11)
    c, n = 6, 20000
    g = rng.normal(0, 3000, (c, n)).astype(np.float16)
    g[2, 17], g[4, 99], g[1, 5] = np.inf, np.nan, -np.inf
    a = g[0].astype(np.float32)
    for k in range(1, c):
        a = (a + g[k].astype(np.float32)).astype(np.float32)
    ref = a.astype(np.float16)
    got = O.accumulate([g[k].view(np.uint16) for k in range(c)], fp32=True)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got.view(np.float16)), nan)
    assert np.array_equal(got[~nan], ref.view(np.uint16)[~nan])


def test_accumulate_fp32_variant_special_cases():
    """What the fp32 accumulator changes, worked by hand: an fp16 partial-sum overflow that cancels later
    (40000 + 40000 - 29984: inf in fp16, 50016 in fp32); a sum reaching 65520 (rounds to inf in either);
    small addends lost in fp16 but kept in fp32 (2048 + 1 + 1 = 2048 in fp16, 2050 in fp32); c = 1 is g_1."""
    h = lambda *v: [np.asarray([x], dtype=np.float16).view(np.uint16) for x in v]  # noqa: E731
    f16 = lambda a: float(a.view(np.float16)[0])  # noqa: E731
    assert np.isinf(f16(O.accumulate(h(40000, 40000, -29984))))
    assert f16(O.accumulate(h(40000, 40000, -29984), fp32=True)) == 50016.0
    assert f16(O.accumulate(h(40000, 40000, -30000), fp32=True)) == 49984.0    # 50000: a tie, to even
    assert np.isinf(f16(O.accumulate(h(32768, 32752), fp32=True)))      # 65520 rounds to inf (R4)
    assert f16(O.accumulate(h(32768, 32736), fp32=True)) == 65504.0      # the largest finite
    assert f16(O.accumulate(h(2048, 1, 1))) == 2048.0
    assert f16(O.accumulate(h(2048, 1, 1), fp32=True)) == 2050.0
    x = np.random.default_rng(2).normal(0, 100, 1000).astype(np.float16).view(np.uint16)
    assert np.array_equal(O.accumulate([x], fp32=True), x)


def test_reduce_spec_examples():
    one = lambda v: np.asarray(v, dtype=np.float16).view(np.uint16)  # noqa: E731
    x = one([1.5, -2.0, 7.0])
    assert np.array_equal(O.reduce([x]), x)                                   # S:391 W=1 identity
    assert np.array_equal(O.reduce([one([1, 2]), one([3, 4])]), one([4, 6]))


def test_reduce_order_dependence_is_real():
    # Reading R3: the oracle fixes ascending rank order because fp16 sums are order dependent.
    h = lambda v: int(np.float16(v).view(np.uint16))  # noqa: E731
    assert O.hadd(O.hadd(h(2048), h(1)), h(1)) == h(2048)
    assert O.hadd(h(2048), O.hadd(h(1), h(1))) == h(2050)
    assert (O.hadd(h(40000), h(40000)) & 0x7C00) == 0x7C00


def test_exact_family_reduce_equals_integer_sum():
    wl = models.Workload("t", [("w", 3000, 0), ("b", 100, 1), ("e", 900, 2)], world=4, update_freq=2,
                         family="exact")
    lay = synth.Layout(wl)
    accs = [O.accumulate([synth.micro_grad_cpu(wl, lay, 1, r, k, 7) for k in (1, 2)]) for r in range(4)]
    R = O.h2d_array(O.reduce(accs))
    exact = sum(synth.micro_grad_cpu(wl, lay, 1, r, k, 7).view(np.float16).astype(np.float64)
                for r in range(4) for k in (1, 2))
    assert np.array_equal(R, exact)


# ============================================================================ LR schedule
def test_lr_golden(gold):
    for t, peak, exp, *_ in gold("lr_schedule.txt"):
        assert O.lr_at(int(t), float(peak)) == np.float32(float(exp)), (t, peak)


def test_lr_shape():
    lr = np.array([O.lr_at(t) for t in range(1, 20001)], dtype=np.float64)
    assert np.all(np.diff(lr[:4000]) > 0)                      # linear warmup
    assert np.all(np.diff(lr[3999:]) < 0)                      # strictly decreasing after
    assert lr[3999] == np.float32(5e-4)                        # continuous at 4000
    t = np.arange(1, 4001)
    assert np.allclose(lr[:4000], 5e-4 * t / 4000, rtol=1e-7, atol=0)
    t = np.arange(4000, 20001)
    assert np.allclose(lr[3999:], 5e-4 * np.sqrt(4000 / t), rtol=1e-7, atol=0)
    assert abs(lr[:100].sum() - 6.3125e-4) < 1e-10           # sum_{t<=100} t/4000*5e-4 = 6.3125e-4


# ============================================================================ scaler
def _step(e, clean, t, overflow, cfg=None):
    cfg = cfg or O.Config()
    s = O.OrcScaler(e, clean, t)
    r = O.OrcResult()
    import ctypes
    O.lib().orc_scaler_step(ctypes.byref(s), ctypes.byref(cfg.c()), int(overflow), ctypes.byref(r))
    return s, r


def test_scaler_golden(gold):
    for ein, cin, ov, eout, cout, app, *_ in gold("scaler_examples.txt"):
        s, r = _step(int(ein), int(cin), 0, int(ov))
        assert (s.e, s.clean, r.applied) == (int(eout), int(cout), int(app))
        assert r.e_used == int(ein) and r.e_next == int(eout)


def test_scaler_matches_torch_amp_update_scale():
    # torch._amp_update_scale_ implements the same state machine (growth after `interval` clean steps,
    # halve on inf); compared on random overflow sequences away from the clamp bounds.
    rng = np.random.default_rng(4)
    interval = 7
    cfg = O.Config(growth=interval)
    for _ in range(20):
        e, clean, t = 7, 0, 0
        scale = torch.tensor([128.0])
        tracker = torch.tensor([0], dtype=torch.int32)
        for ov in rng.random(200) < 0.08:
            s, r = _step(e, clean, t, ov, cfg)
            e, clean, t = s.e, s.clean, s.t
            torch._amp_update_scale_(scale, tracker, torch.tensor([float(ov)]), 2.0, 0.5, interval)
            assert scale.item() == 2.0 ** e and tracker.item() == clean
            assert -5 < e < 24


def test_scaler_trace_closed_forms(gold):
    # C0 (BASELINE configs[0]) per-update trace and C3 checkpoints, derived by hand from P:156-158.
    s = O.OrcScaler(7, 0, 0)
    cfg = O.Config().c()
    import ctypes
    for u, ov, app, eu, en, t, clean, lrs in (map(int, r) for r in gold("scaler_trace_c0.txt")):
        r = O.OrcResult()
        O.lib().orc_scaler_step(ctypes.byref(s), ctypes.byref(cfg), ov, ctypes.byref(r))
        assert (r.overflow, r.applied, r.e_used, r.e_next, r.t, r.clean) == (ov, app, eu, en, t, clean), u
        assert r.lr == O.lr_at(lrs)
    s = O.OrcScaler(7, 0, 0)
    burst = set(range(2500, 2504)) | set(range(5000, 5004))
    checks = {int(r[0]): tuple(map(int, r[1:])) for r in gold("scaler_trace_c3.txt")}
    for u in range(1, 5201):
        r = O.OrcResult()
        O.lib().orc_scaler_step(ctypes.byref(s), ctypes.byref(cfg), int(u in burst), ctypes.byref(r))
        if u in checks:
            assert (s.e, s.clean, s.t) == checks[u], u


# ============================================================================ Adam
def _adam_once(R16, e, N, lr, t, theta, m=None, v=None, cfg=None):
    cfg = cfg or O.Config()
    n = len(R16)
    th = np.asarray(theta, dtype=np.float64).copy()
    m = np.zeros(n) if m is None else m.copy()
    v = np.zeros(n) if v is None else v.copy()
    w = np.zeros(n, dtype=np.uint16)
    R = np.ascontiguousarray(R16, dtype=np.uint16)
    import ctypes
    O.lib().orc_adam(O._p(th), O._p(m), O._p(v), O._p(w), O._p(R), n, e, N, lr, t, ctypes.byref(cfg.c()))
    return th, m, v, w


def test_adam_spec_first_step():
    # first step, g = 1, lr = 1e-3 -> dtheta = -1e-3 * 1/(1 + 1e-8) ~ -9.99999990e-4
    lr = np.float32(1e-3)
    th, m, v, w = _adam_once([0x3C00], 0, 1, lr, 1, [0.0])
    assert th[0] == pytest.approx(-float(lr) / (1 + 1e-8), rel=1e-15)
    assert th[0] == pytest.approx(-9.99999990e-4, rel=1e-7)
    assert m[0] == pytest.approx(0.1, rel=1e-15) and v[0] == pytest.approx(0.02, rel=1e-15)
    assert w[0] == np.float16(th[0]).view(np.uint16)


def test_adam_zero_gradient_is_identity():
    # g = 0 everywhere, fresh state -> params unchanged, moments exactly 0
    theta = np.array([0.5, -1.25, 3.0])
    th, m, v, w = _adam_once([0, 0, 0x8000], 7, 1000, np.float32(1e-3), 1, theta)
    assert np.array_equal(th, theta) and not m.any() and not v.any()


def test_adam_constant_gradient_closed_form():
    # m_hat_t = g and v_hat_t = g^2 for constant g => theta_T = theta_0 - g/(|g|+eps) * sum_t lr_t
    g16 = np.float16(0.375).view(np.uint16)
    e, N = 3, 2
    g = 0.375 / (2**e * N)
    th, m, v = np.array([0.25]), np.zeros(1), np.zeros(1)
    lrsum = 0.0
    for t in range(1, 101):
        lr = O.lr_at(t)
        lrsum += float(lr)
        th, m, v, _ = _adam_once([g16], e, N, lr, t, th, m, v)
    assert th[0] == pytest.approx(0.25 - g / (abs(g) + 1e-8) * lrsum, rel=1e-12)


def test_adam_matches_torch_optim_adam_fp64():
    rng = np.random.default_rng(5)
    n, e = 257, 5
    theta0 = rng.normal(0, 0.1, n)
    p = torch.nn.Parameter(torch.tensor(theta0, dtype=torch.float64))
    opt = torch.optim.Adam([p], lr=1.0, betas=(0.9, 0.98), eps=1e-8, foreach=False, fused=False)
    th, m, v = theta0.copy(), np.zeros(n), np.zeros(n)
    for t in range(1, 101):
        R = rng.normal(0, 8, n).astype(np.float16).view(np.uint16)
        N = int(rng.integers(1000, 5000))
        lr = O.lr_at(t)
        th, m, v, w = _adam_once(R, e, N, lr, t, th, m, v)
        p.grad = torch.tensor(R.view(np.float16).astype(np.float64) / (2**e * N))
        for grp in opt.param_groups:
            grp["lr"] = float(lr)
        opt.step()
    assert np.allclose(th, p.detach().numpy(), rtol=1e-12, atol=1e-15)
    st = opt.state[p]
    assert np.allclose(m, st["exp_avg"].numpy(), rtol=1e-12, atol=0)
    assert np.allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-12, atol=0)
    assert np.array_equal(w, th.astype(np.float16).view(np.uint16))


# ============================================================================ whole update
def test_skip_leaves_state_unchanged():
    wl = models.tiny(updates=3, injections=[dict(u=2, kind="NAN", r=0, k=1, i=10)])
    orc, trace = O.run_workload(wl, 1)
    before = (orc.theta.copy(), orc.m.copy(), orc.v.copy(), orc.w16.copy(), orc.s.t)
    lay = synth.Layout(wl)
    grads = [[synth.micro_grad_cpu(wl, lay, 2, 0, k, orc.e) for k in (1, 2)]]
    res = orc.update(grads, [[3000, 3000]])
    assert res["overflow"] == 1 and res["applied"] == 0 and res["e_next"] == 6
    assert np.array_equal(orc.theta, before[0]) and np.array_equal(orc.m, before[1])
    assert np.array_equal(orc.v, before[2]) and np.array_equal(orc.w16, before[3]) and orc.s.t == before[4]


@pytest.mark.parametrize("kind", ["INF", "NINF", "NAN", "ACC_OVF"])
def test_injection_kinds_overflow(kind):
    inj = [dict(u=1, kind=kind, r=0, k=2, i=77)]
    wl = models.Workload("t", [("w", 2000, 0)], 1, 2, injections=inj)
    _, trace = O.run_workload(wl, 1)
    assert trace[0]["overflow"] == 1 and trace[0]["applied"] == 0


def test_red_ovf_overflows_only_after_reduce():
    wl = models.Workload("t", [("w", 2000, 0)], 2, 2, injections=[dict(u=1, kind="RED_OVF", i=5)])
    lay = synth.Layout(wl)
    accs = [O.accumulate([synth.micro_grad_cpu(wl, lay, 1, r, k, 7) for k in (1, 2)]) for r in range(2)]
    assert all(O.count_nonfinite(a) == 0 for a in accs)        # locally finite on every rank
    assert O.count_nonfinite(O.reduce(accs)) == 1              # 40000 + 40000 -> +inf after the sum


def test_tiny_trace_matches_closed_form(gold):
    wl = models.tiny()
    _, trace = O.run_workload(wl, 10)
    for res, row in zip(trace, gold("scaler_trace_c0.txt")):
        u, ov, app, eu, en, t, clean, lrs = map(int, row)
        assert (res["overflow"], res["applied"], res["e_used"], res["e_next"], res["t"], res["clean"]) == \
               (ov, app, eu, en, t, clean)
        assert res["lr"] == O.lr_at(lrs)


def test_world_and_accumulation_equivalence_exact_family():
    # SPEC S:400-401 / S:437: (W, c) groupings of the same 8 exactly-summable micro-gradients give
    # bitwise identical state (G_exact, reading R3).  The micro set is fixed: micro j of the global set is
    # (u, r = j // c, k = j % c + 1) of the (W=1, c=8) numbering.
    base = models.Workload("t", [("w", 3000, 0), ("b", 64, 1)], 1, 8, family="exact")
    lay = synth.Layout(base)
    micro = [synth.micro_grad_cpu(base, lay, 1, 0, k, 7) for k in range(1, 9)]
    ref = None
    for W, c in ((1, 8), (2, 4), (4, 2), (8, 1)):
        orc = O.Oracle(synth.theta0_cpu(base, lay))
        grads = [[micro[r * c + k] for k in range(c)] for r in range(W)]
        orc.update(grads, [[100] * c for _ in range(W)])
        state = (orc.theta, orc.m, orc.v, orc.w16)
        if ref is None:
            ref = state
        else:
            for a, b in zip(ref, state):
                assert np.array_equal(a, b), (W, c)


def test_one_rank_many_micro_equals_many_ranks_one_micro_real_values():
    # SURVEY c.3: with G_real (order-dependent values) only (W=1, c) == (W=c, 1) holds bitwise -- the same
    # association: ((g1 + g2) + g3) + g4 locally, or ascending-rank ((A0 + A1) + A2) + A3.
    base = models.Workload("t", [("w", 20_000, 0), ("e", 999, 2)], 1, 4)
    lay = synth.Layout(base)
    micro = [synth.micro_grad_cpu(base, lay, 1, 0, k, 7) for k in range(1, 5)]
    states = []
    for W, c in ((1, 4), (4, 1)):
        orc = O.Oracle(synth.theta0_cpu(base, lay))
        orc.update([[micro[r * c + k] for k in range(c)] for r in range(W)], [[10] * c for _ in range(W)])
        states.append((orc.theta, orc.m, orc.v, orc.w16))
    for a, b in zip(*states):
        assert np.array_equal(a, b)
    # and a regrouping with a different association is NOT bitwise in general (SPEC S:633's claim is false)
    orc = O.Oracle(synth.theta0_cpu(base, lay))
    res = orc.update([[micro[0], micro[1]], [micro[2], micro[3]]], [[10, 10], [10, 10]])
    ref = O.reduce([O.accumulate(micro)])
    assert not np.array_equal(res["R"], ref)


def test_large_batch_gradient_softmax_regression():
    # North star pin: the summed micro-batch gradient equals the single-worker large-batch gradient, and
    # the update divides it once by the global target-token count N.  Brute force on a tiny
    # softmax regression (V=7 classes, d=5 features, 4 micro-batches) in fp64.
    rng = np.random.default_rng(6)
    V, d = 7, 5
    Wt = rng.normal(0, 0.5, (V, d))

    def grad_sum(X, y):     # d/dW of the token-SUM cross-entropy
        z = X @ Wt.T
        p = np.exp(z - z.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        p[np.arange(len(y)), y] -= 1.0
        return p.T @ X

    batches = [(rng.normal(0, 1, (nb, d)), rng.integers(0, V, nb)) for nb in (5, 9, 3, 7)]
    gs = [grad_sum(X, y) for X, y in batches]
    Xc = np.concatenate([b[0] for b in batches])
    yc = np.concatenate([b[1] for b in batches])
    assert np.allclose(sum(gs), grad_sum(Xc, yc), rtol=1e-12, atol=1e-12)
    # finite-difference check of the analytic gradient itself
    eps = 1e-6

    def loss(Wm):
        z = Xc @ Wm.T
        return float((np.log(np.exp(z).sum(1)) - z[np.arange(len(yc)), yc]).sum())
    fd = np.zeros_like(Wt)
    for i in range(V):
        for j in range(d):
            Wp, Wm_ = Wt.copy(), Wt.copy()
            Wp[i, j] += eps
            Wm_[i, j] -= eps
            fd[i, j] = (loss(Wp) - loss(Wm_)) / (2 * eps)
    assert np.allclose(fd, grad_sum(Xc, yc), rtol=1e-6, atol=1e-7)
    # push scaled fp16 micro-gradients through the oracle (W=2, c=2) and read g back out of m after step 1
    orc = O.Oracle(np.zeros(V * d, dtype=np.float32))
    e = orc.e                    # the producer scales the loss by the library's current 2^e
    micro = [np.asarray(g.ravel() * 2.0**e, dtype=np.float16).view(np.uint16) for g in gs]
    N = len(yc)
    res = orc.update([[micro[0], micro[1]], [micro[2], micro[3]]], [[5, 9], [3, 7]])
    assert res["applied"] == 1 and res["N"] == N
    g_oracle = orc.m / (1 - 0.9)
    g_true = (grad_sum(Xc, yc) / N).ravel()
    # fp16 quantisation bound: 7 roundings (4 micro-gradients, 2 local adds, 1 cross-rank add), each at
    # most 2^-11 of a magnitude <= sum_k |g_k| (plus the subnormal quantum 2^-24 before unscaling).
    mag = sum(np.abs(g.ravel()) for g in gs) / N
    bound = 7 * (2.0**-11 * mag + 2.0**-24 / (2.0**e * N))
    assert np.all(np.abs(g_oracle - g_true) <= bound)
    # and the normalisation is by N exactly: a wrong divisor (N_r, c, W, or a dropped 2^e) misses by >= 2x
    assert np.abs(g_oracle - g_true).max() < 0.01 * np.abs(g_true).max()


def test_c_whole_update_equals_python_driver():
    # oracle.c's orc_update (the c.1 body in one C call) and the Python driver's step-by-step calls agree
    import ctypes
    wl = models.Workload("t", [("w", 5000, 0), ("b", 33, 1)], 3, 2, injections=[dict(u=2, kind="INF", r=1, k=2, i=7)])
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    py = O.Oracle(theta0)
    n = lay.n
    th = theta0.astype(np.float64)
    m, v = np.zeros(n), np.zeros(n)
    w16 = O.d2h_array(th)
    s = O.OrcScaler(7, 0, 0)
    A = np.empty(3 * n, np.uint16)
    R = np.empty(n, np.uint16)
    for u in (1, 2, 3):
        grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, s.e) for k in (1, 2)] for r in range(3)]
        toks = [[100 * (r + 1), 50] for r in range(3)]
        rp = py.update(grads, toks)
        flat = [g for row in grads for g in row]
        arr = (ctypes.c_void_p * len(flat))(*[g.ctypes.data for g in flat])
        res = O.OrcResult()
        N = sum(sum(t) for t in toks)
        O.lib().orc_update(O._p(th), O._p(m), O._p(v), O._p(w16), n, arr, 3, 2, N, O._p(A), O._p(R), ctypes.byref(s),
                           ctypes.byref(O.Config().c()), ctypes.byref(res))
        assert res.as_dict() == {k: rp[k] for k in res.as_dict()}, u
        assert np.array_equal(R, rp["R"])
        assert np.array_equal(th, py.theta) and np.array_equal(m, py.m) and np.array_equal(v, py.v)
        assert np.array_equal(w16, py.w16)
