"""Python driver for the CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only permitted callers.  Nothing
in paper_1806_00187_b200/ imports this module.

The driver is a plain transcription of SURVEY.md 8(c.1) (itself PAPER.md 4.1-4.3
and 3.2): per update, generate the W*c micro-gradients (synth/, inputs only),
accumulate per rank, reduce in ascending rank order, test for overflow, run the
scaler and, when clean, Adam in fp64.  Element arithmetic runs in oracle.c.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


class OrcCfg(ctypes.Structure):
    _fields_ = [("peak_lr", ctypes.c_double), ("warmup", ctypes.c_int64), ("beta1", ctypes.c_double),
                ("beta2", ctypes.c_double), ("eps", ctypes.c_double), ("emin", ctypes.c_int32),
                ("emax", ctypes.c_int32), ("growth", ctypes.c_int64)]


class OrcScaler(ctypes.Structure):
    _fields_ = [("e", ctypes.c_int32), ("clean", ctypes.c_int64), ("t", ctypes.c_int64)]


class OrcResult(ctypes.Structure):
    _fields_ = [("overflow", ctypes.c_int32), ("applied", ctypes.c_int32), ("e_used", ctypes.c_int32),
                ("e_next", ctypes.c_int32), ("lr", ctypes.c_float), ("t", ctypes.c_int64),
                ("N", ctypes.c_int64), ("clean", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        p, i64, i32, u16, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint16, ctypes.c_double
        L.orc_h2d.restype = d
        L.orc_h2d.argtypes = [u16]
        L.orc_d2h.restype = u16
        L.orc_d2h.argtypes = [d]
        L.orc_hadd.restype = u16
        L.orc_hadd.argtypes = [u16, u16]
        L.orc_h_nonfinite.restype = i32
        L.orc_h_nonfinite.argtypes = [u16]
        L.orc_h2d_array.argtypes = [p, p, i64]
        L.orc_d2h_array.argtypes = [p, p, i64]
        L.orc_set_threads.restype = i32
        L.orc_set_threads.argtypes = [i32]
        L.orc_accumulate.argtypes = [p, p, i64, i32]
        L.orc_accumulate32.argtypes = [p, p, i64, i32]
        L.orc_round16.argtypes = [p, p, i64]
        L.orc_reduce.argtypes = [p, p, i32, i64]
        L.orc_count_nonfinite.restype = i64
        L.orc_count_nonfinite.argtypes = [p, i64]
        L.orc_lr.restype = ctypes.c_float
        L.orc_lr.argtypes = [i64, d, i64]
        L.orc_scaler_step.restype = i32
        L.orc_scaler_step.argtypes = [ctypes.POINTER(OrcScaler), ctypes.POINTER(OrcCfg), i32,
                                      ctypes.POINTER(OrcResult)]
        L.orc_adam.argtypes = [p, p, p, p, p, i64, ctypes.c_int32, i64, ctypes.c_float, i64,
                               ctypes.POINTER(OrcCfg)]
        L.orc_update.restype = i32
        L.orc_update.argtypes = [p, p, p, p, i64, p, i32, i32, i64, p, p, ctypes.POINTER(OrcScaler),
                                 ctypes.POINTER(OrcCfg), ctypes.POINTER(OrcResult)]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


# ----------------------------------------------------------------------------- scalar helpers
def h2d(bits: int) -> float:
    return lib().orc_h2d(bits)


def d2h(x: float) -> int:
    return lib().orc_d2h(x)


def hadd(a: int, b: int) -> int:
    return lib().orc_hadd(a, b)


def h2d_array(h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16)
    out = np.empty(h.size, dtype=np.float64)
    lib().orc_h2d_array(_p(h), _p(out), h.size)
    return out


def d2h_array(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.size, dtype=np.uint16)
    lib().orc_d2h_array(_p(x), _p(out), x.size)
    return out


def set_threads(t: int) -> int:
    """OpenMP threads of the oracle's element loops (t <= 0: query); returns the count in effect."""
    return lib().orc_set_threads(t)


def lr_at(t: int, peak: float = 5e-4, warmup: int = 4000) -> float:
    return lib().orc_lr(t, peak, warmup)


def accumulate(grads, fp32: bool = False) -> np.ndarray:
    """A = g_1, then A = rn16(A + g_k).  fp32: the Z1 variant, A32 = fp32(g_1), A32 = fl32(A32 + g_k),
    returned as rn16(A32) (oracle.c orc_accumulate32)."""
    if fp32:
        A32 = np.empty(np.asarray(grads[0]).size, dtype=np.float32)
        for k, g in enumerate(grads):
            g = np.ascontiguousarray(g, dtype=np.uint16)
            lib().orc_accumulate32(_p(A32), _p(g), A32.size, 1 if k == 0 else 0)
        A = np.empty(A32.size, dtype=np.uint16)
        lib().orc_round16(_p(A), _p(A32), A32.size)
        return A
    A = np.empty_like(grads[0])
    for k, g in enumerate(grads):
        g = np.ascontiguousarray(g, dtype=np.uint16)
        lib().orc_accumulate(_p(A), _p(g), A.size, 1 if k == 0 else 0)
    return A


def reduce(accs) -> np.ndarray:
    """R = A_0 + A_1 + ... in ascending rank order, rn16 per add (reading R3)."""
    accs = [np.ascontiguousarray(a, dtype=np.uint16) for a in accs]
    R = np.empty_like(accs[0])
    arr = (ctypes.c_void_p * len(accs))(*[a.ctypes.data for a in accs])
    lib().orc_reduce(_p(R), arr, len(accs), R.size)
    return R


def count_nonfinite(R: np.ndarray) -> int:
    R = np.ascontiguousarray(R, dtype=np.uint16)
    return lib().orc_count_nonfinite(_p(R), R.size)


# ----------------------------------------------------------------------------- stateful oracle
@dataclass
class Config:
    peak_lr: float = 5e-4        # P:105 (1e-3 for "2x lr")
    warmup: int = 4000
    beta1: float = 0.9
    beta2: float = 0.98
    eps: float = 1e-8
    init_scale_log2: int = 7     # reading R8
    min_scale_log2: int = -5
    max_scale_log2: int = 24
    growth: int = 2000
    accum_fp32: bool = False     # SURVEY Z1 knob: fp32 accumulator, rn16 before the fp16 all-reduce

    def c(self):
        return OrcCfg(self.peak_lr, self.warmup, self.beta1, self.beta2, self.eps, self.min_scale_log2,
                      self.max_scale_log2, self.growth)


class Oracle:
    """State of SURVEY 8(c.1): theta, m, v in fp64; w16 binary16; scaler (e, clean, t).

    `theta0` may be the full fp32 vector or a sample of it (sampled parity: every
    stage but the overflow decision is elementwise, so the state at sampled indices
    is exact given the decision, which the caller then supplies from a full pass)."""

    def __init__(self, theta0: np.ndarray, cfg: Config | None = None):
        self.cfg = cfg or Config()
        self._c = self.cfg.c()
        self.theta = np.ascontiguousarray(theta0, dtype=np.float32).astype(np.float64)
        self.m = np.zeros_like(self.theta)
        self.v = np.zeros_like(self.theta)
        self.w16 = d2h_array(self.theta)
        self.s = OrcScaler(self.cfg.init_scale_log2, 0, 0)

    @property
    def e(self):
        return self.s.e

    def update(self, grads, ntokens, overflow: bool | None = None) -> dict:
        """grads[r][k]: uint16 arrays (same index set as theta); ntokens[r][k]: ints.

        overflow=None: decide from these arrays (full-vector mode).  Otherwise the caller's
        full-vector decision is used (sampled mode)."""
        W, c = len(grads), len(grads[0])
        N = int(sum(sum(row) for row in ntokens))
        A = [accumulate(grads[r], self.cfg.accum_fp32) for r in range(W)]
        R = reduce(A)
        if overflow is None:
            overflow = count_nonfinite(R) > 0
        res = OrcResult()
        e_used = self.s.e
        res.N = N
        if N == 0:
            raise ValueError("N = 0: update discarded (reading R19)")
        applied = lib().orc_scaler_step(ctypes.byref(self.s), ctypes.byref(self._c), int(bool(overflow)),
                                        ctypes.byref(res))
        if applied:
            lib().orc_adam(_p(self.theta), _p(self.m), _p(self.v), _p(self.w16), _p(R), R.size, e_used, N,
                           res.lr, self.s.t, ctypes.byref(self._c))
        out = res.as_dict()
        out["R"] = R
        return out

    def scaler_state(self):
        return dict(e=self.s.e, clean=self.s.clean, t=self.s.t)


# ----------------------------------------------------------------------------- workload drivers
def full_overflow(wl, lay, u: int, e: int, chunk: int = 1 << 22, accum_fp32: bool = False) -> bool:
    """Overflow decision of update u over the FULL vector, streamed in index chunks."""
    import synth
    W, c = wl.world, wl.update_freq
    for lo in range(0, lay.n, chunk):
        hi = min(lay.n, lo + chunk)
        accs = [accumulate([synth.micro_grad_range(wl, lay, lo, hi, u, r, k, e) for k in range(1, c + 1)],
                           accum_fp32) for r in range(W)]
        if count_nonfinite(reduce(accs)) > 0:
            return True
    return False


def run_workload(wl, updates: int, idx: np.ndarray | None = None, decisions_full: bool = True,
                 cfg: Config | None = None, record=None):
    """Run the oracle over `updates` updates of workload wl.

    idx=None: full vectors.  Otherwise state is kept only at idx; the overflow
    decision is taken over the full vector when decisions_full (streamed), else it
    is the injection schedule's (every update with an injection overflows; the
    bounded generators cannot overflow by themselves)."""
    import synth
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay) if idx is None else synth.theta0_sample(wl, idx)
    orc = Oracle(theta0, cfg)
    trace = []
    inj_updates = {inj["u"] for inj in wl.injections}
    for u in range(1, updates + 1):
        e = orc.e
        W, c = wl.world, wl.update_freq
        if idx is None:
            grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, e) for k in range(1, c + 1)] for r in range(W)]
            ov = None
        else:
            grads = [[synth.micro_grad_sample(wl, lay, idx, u, r, k, e) for k in range(1, c + 1)] for r in range(W)]
            ov = full_overflow(wl, lay, u, e) if decisions_full else (u in inj_updates)
        toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(W)]
        res = orc.update(grads, toks, overflow=ov)
        res.pop("R")
        trace.append(res)
        if record is not None:
            record(u, orc)
    return orc, trace
