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
    from paper_1806_00187_b200 import smpu
    ocfg = ocfg or O.Config()
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


class Magnitudes:
    """Cancellation-safe operand scales for accumulated state (reading R26, refining SURVEY 8(c.4)):
    theta: |theta_0| + sum_t |dtheta_t|;  m: EMA of |g| (mag_m = b1 mag_m + (1-b1)|g|);  v: |v| (sum of
    non-negative terms).  A relative error measured against these bounds what fp32 rounding of every term that
    ever entered the value can produce, which a one-step operand scale cannot when a value cancels to ~0."""

    def __init__(self, theta0):
        self.th = np.abs(np.asarray(theta0, dtype=np.float64))
        self.m = np.zeros_like(self.th)

    def update(self, R16, e, N, th_before, th_after):
        g = np.abs(O.h2d_array(R16)) / (2.0**e * N)
        self.m = B1 * self.m + (1 - B1) * g
        self.th = self.th + np.abs(th_after - th_before)


def check_state(gpu, orc_now, mags, rtol, where=""):
    """gpu: dict theta/m/v (fp32) + w16 (uint16) at the oracle's index set; orc_now: oracle snapshot (fp64);
    mags: Magnitudes at the same indices.  |x_gpu - x_ref| <= rtol * D, exact zeros exact, w16 within 1 ulp."""
    th, m, v = orc_now["theta"], orc_now["m"], orc_now["v"]
    for name, ref, D in (("theta", th, mags.th), ("m", m, mags.m), ("v", v, np.abs(v))):
        x = gpu[name].astype(np.float64)
        zero = ref == 0
        assert np.array_equal(x[zero], ref[zero]), f"{where}: {name} exact zeros differ"
        err = np.abs(x - ref)
        bad = err > rtol * D
        assert not bad.any(), (f"{where}: {name} {bad.sum()} elements beyond {rtol} (worst at "
                               f"{int(np.argmax(err / np.maximum(D, 1e-300)))}: gpu {x[bad][:3]} ref {ref[bad][:3]})")
    d = ulp16_dist(gpu["w16"], orc_now["w16"])
    assert d.max() <= 1, f"{where}: w16 differs by {d.max()} ulp"


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
