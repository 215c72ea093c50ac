"""Helpers for the GPU parity tests: drive libsmpu.so (through its binding) and the oracle side by side."""
from __future__ import annotations

import numpy as np

import oracle as O
import synth

B1, B2 = 0.9, 0.98

# SURVEY 8(c.4) tolerances (north_star): theta/m/v 1e-6 relative after 1 update, 1e-4 after 100.
RTOL_1 = 1e-6
RTOL_100 = 1e-4


def lib_cfg(wl, ocfg: O.Config | None = None, **kw):
    """The library config of a test workload.  fuse_final defaults to 1 HERE (the library's default is 0) so that the
    runners keep exercising the fused last micro-batch beside the explicit fuse_final = 0 ctxs they compare with."""
    from paper_1806_00187_b200 import smpu
    ocfg = ocfg or O.Config()
    kw.setdefault("fuse_final", 1)
    c = smpu.config_default(peak_lr=ocfg.peak_lr, warmup_updates=ocfg.warmup, beta1=ocfg.beta1, beta2=ocfg.beta2,
                            eps=ocfg.eps, init_scale_log2=ocfg.init_scale_log2, min_scale_log2=ocfg.min_scale_log2,
                            max_scale_log2=ocfg.max_scale_log2, growth_interval=ocfg.growth,
                            update_freq=wl.update_freq, accum_fp32=int(ocfg.accum_fp32))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def decisions(res: dict):
    """The bitwise-compared decision tuple of one update (c.4), library result dict."""
    return (res["overflow"], res["applied"], res["scale_log2_used"], res["scale_log2_next"],
            np.float32(res["lr"]).view(np.uint32).item(), res["num_updates"], res["ntokens_total"],
            res["clean_streak"])


def oracle_decisions(res: dict):
    return (res["overflow"], res["applied"], res["e_used"], res["e_next"],
            np.float32(res["lr"]).view(np.uint32).item(), res["t"], res["N"], res["clean"])


def ulp16_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|key(a) - key(b)| with key(h) = +(h & 0x7FFF) for sign 0, -(h & 0x7FFF) for sign 1 (c.4)."""
    def key(h):
        h = h.astype(np.int64)
        mag = h & 0x7FFF
        return np.where(h & 0x8000, -mag, mag)
    return np.abs(key(a) - key(b))


def rtol_for(t: int) -> float:
    """Tolerance on theta/m/v after t applied updates: the north star's 1e-6 after 1 update and 1e-4 after 100
    (SURVEY 8(c.4)), joined linearly -- an error budget of 1e-6 per applied update, capped at 1e-4 (reading R28)."""
    return min(RTOL_100, RTOL_1 * max(int(t), 1))


class Magnitudes:
    """Operand scales D of the parity check.

    R26 (cumulative, the asserted one): theta: |theta_0| + sum_t |dtheta_t|;  m: EMA of |g|
    (mag_m = b1 mag_m + (1-b1)|g|);  v: |v| (sum of non-negative terms).  A relative error against these bounds what
    fp32 rounding of every term that ever entered the value can produce, which a one-step scale cannot when a value
    cancels to ~0.
    SURVEY 8(c.4) one-step D (reported beside it): theta: max(|theta_ref|, |theta_prev| + |dtheta|);
    m: max(|m_ref|, b1|m_prev| + (1-b1)|g|);  v: |v_ref|.  Identical to R26's after the first update."""

    def __init__(self, theta0):
        self.th = np.abs(np.asarray(theta0, dtype=np.float64))
        self.m = np.zeros_like(self.th)
        self.th1 = self.th.copy()          # one-step D (c.4), theta
        self.m1 = np.zeros_like(self.th)   # one-step D (c.4), m (without the |m_ref| term, added at check time)

    def update(self, R16, e, N, th_before, th_after, m_before=None):
        g = np.abs(O.h2d_array(R16)) / (2.0**e * N)
        self.m = B1 * self.m + (1 - B1) * g
        self.th = self.th + np.abs(th_after - th_before)
        self.th1 = np.abs(th_before) + np.abs(th_after - th_before)
        mb = np.zeros_like(g) if m_before is None else np.abs(np.asarray(m_before, dtype=np.float64))
        self.m1 = B1 * mb + (1 - B1) * g


def check_state(gpu, orc_now, mags, rtol, where="", report=None):
    """gpu: dict theta/m/v (fp32) + w16 (uint16) at the oracle's index set; orc_now: oracle snapshot (fp64);
    mags: Magnitudes at the same indices.  Asserts |x_gpu - x_ref| <= rtol * D (R26's D), exact zeros exact, w16
    within 1 ulp.  Returns (and appends to `report`, if a list) the worst err/D under R26's D and under SURVEY
    8(c.4)'s one-step D, per array, plus the plain relative error's max and 99.99th percentile."""
    th, m, v = orc_now["theta"], orc_now["m"], orc_now["v"]
    out = {"where": where, "rtol": rtol}
    for name, ref, D, D1 in (("theta", th, mags.th, np.maximum(np.abs(th), mags.th1)),
                             ("m", m, mags.m, np.maximum(np.abs(m), mags.m1)), ("v", v, np.abs(v), np.abs(v))):
        x = gpu[name].astype(np.float64)
        zero = ref == 0
        assert np.array_equal(x[zero], ref[zero]), f"{where}: {name} exact zeros differ"
        err = np.abs(x - ref)
        nz = ~zero
        plain = err[nz] / np.abs(ref[nz]) if nz.any() else np.zeros(1)
        out[name] = {"r26": float(np.max(err / np.maximum(D, 1e-300), initial=0.0)),
                     "c4": float(np.max(err / np.maximum(D1, 1e-300), initial=0.0)),
                     "plain_max": float(plain.max(initial=0.0)),
                     "plain_p9999": float(np.percentile(plain, 99.99)) if plain.size else 0.0}
        bad = err > rtol * D
        assert not bad.any(), (f"{where}: {name} {bad.sum()} elements beyond {rtol} (worst at "
                               f"{int(np.argmax(err / np.maximum(D, 1e-300)))}: gpu {x[bad][:3]} ref {ref[bad][:3]})")
    d = ulp16_dist(gpu["w16"], orc_now["w16"])
    assert d.max(initial=0) <= 1, f"{where}: w16 differs by {d.max()} ulp"
    out["w16_max_ulp"] = int(d.max(initial=0))
    if report is not None:
        report.append(out)
    return out


def format_report(rows) -> str:
    """One line per checked array: worst err/D under R26 and under c.4's one-step D, and the plain rel. error."""
    worst = {}
    for r in rows:
        for name in ("theta", "m", "v"):
            w = worst.setdefault(name, {"r26": 0.0, "c4": 0.0, "plain_max": 0.0, "plain_p9999": 0.0})
            for k in w:
                w[k] = max(w[k], r[name][k])
    return "; ".join(f"{n}: err/D {w['r26']:.2e} (R26) {w['c4']:.2e} (c.4 one-step), plain rel max "
                     f"{w['plain_max']:.2e} p99.99 {w['plain_p9999']:.2e}" for n, w in worst.items())


def snapshot(orc: O.Oracle, idx=None):
    sel = slice(None) if idx is None else idx
    return dict(theta=orc.theta[sel].copy(), m=orc.m[sel].copy(), v=orc.v[sel].copy(), w16=orc.w16[sel].copy())


def gpu_state(step, idx=None):
    from paper_1806_00187_b200 import smpu
    out = {}
    for name, which in (("theta", smpu.STATE_MASTER), ("m", smpu.STATE_M), ("v", smpu.STATE_V),
                        ("w16", smpu.STATE_W16)):
        a = step.get_state(which)
        out[name] = a if idx is None else a[idx]
    return out


def h2t(arr: np.ndarray):
    """uint16 numpy -> int16 cuda tensor (bit copy)."""
    import torch
    return torch.from_numpy(arr.view(np.int16)).cuda()
