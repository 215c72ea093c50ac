"""ctypes binding of libsmpu_sched.so (include/smpu_sched.h): the host-side straggler / batching component
(section 5).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsmpu_sched.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py`")
        L = ctypes.CDLL(LIB_PATH)
        p, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        P = ctypes.POINTER
        L.smpu_sched_token_budget.argtypes = [p, p, i64, i64, p, p, i64, P(ctypes.c_int64)]
        L.smpu_sched_fit_timing.argtypes = [p, p, p, p, i64, p]
        L.smpu_sched_estimate.argtypes = [p, p, p, p, i64, p, p]
        L.smpu_sched_time_balanced.argtypes = [p, p, i64, p, d, p, p, i64, P(ctypes.c_int64)]
        L.smpu_sched_simulate.argtypes = [p, i64, i32, i32, P(ctypes.c_double), P(ctypes.c_double),
                                          P(ctypes.c_int64)]
        L.smpu_sched_overlap_schedule.argtypes = [p, p, i64, d, d, d, i32, p, p, p, p, i64, P(ctypes.c_int64),
                                                  P(ctypes.c_double), P(ctypes.c_double)]
        for f in ("smpu_sched_token_budget", "smpu_sched_fit_timing", "smpu_sched_estimate",
                  "smpu_sched_time_balanced", "smpu_sched_simulate", "smpu_sched_overlap_schedule"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"{what}: status {rc}")


def _lens(src, tgt):
    return np.ascontiguousarray(src, dtype=np.int32), np.ascontiguousarray(tgt, dtype=np.int32)


def token_budget(src, tgt, max_tokens):
    """-> (order, batch_begin): sub-batch b is order[batch_begin[b]:batch_begin[b+1]]."""
    src, tgt = _lens(src, tgt)
    n = src.size
    order = np.zeros(max(n, 1), np.int64)
    begin = np.zeros(n + 2, np.int64)
    nb = ctypes.c_int64()
    _check(lib().smpu_sched_token_budget(_p(src), _p(tgt), n, int(max_tokens), _p(order), _p(begin), n + 1,
                                         ctypes.byref(nb)), "token_budget")
    return order[:n], begin[: nb.value + 1]


def time_balanced(src, tgt, coef, target_seconds):
    src, tgt = _lens(src, tgt)
    n = src.size
    order = np.zeros(max(n, 1), np.int64)
    begin = np.zeros(n + 2, np.int64)
    nb = ctypes.c_int64()
    c = np.ascontiguousarray(coef, dtype=np.float64)
    _check(lib().smpu_sched_time_balanced(_p(src), _p(tgt), n, _p(c), float(target_seconds), _p(order), _p(begin),
                                          n + 1, ctypes.byref(nb)), "time_balanced")
    return order[:n], begin[: nb.value + 1]


def fit_timing(sentences, max_src, max_tgt, seconds):
    s = np.ascontiguousarray(sentences, dtype=np.int32)
    a = np.ascontiguousarray(max_src, dtype=np.int32)
    b = np.ascontiguousarray(max_tgt, dtype=np.int32)
    t = np.ascontiguousarray(seconds, dtype=np.float64)
    coef = np.zeros(3, np.float64)
    _check(lib().smpu_sched_fit_timing(_p(s), _p(a), _p(b), _p(t), s.size, _p(coef)), "fit_timing")
    return coef


def estimate(src, tgt, order, begin, coef):
    src, tgt = _lens(src, tgt)
    order = np.ascontiguousarray(order, dtype=np.int64)
    begin = np.ascontiguousarray(begin, dtype=np.int64)
    c = np.ascontiguousarray(coef, dtype=np.float64)
    out = np.zeros(max(begin.size - 1, 1), np.float64)
    _check(lib().smpu_sched_estimate(_p(src), _p(tgt), _p(order), _p(begin), begin.size - 1, _p(c), _p(out)),
           "estimate")
    return out[: begin.size - 1]


def simulate(batch_seconds, workers, update_freq):
    t = np.ascontiguousarray(batch_seconds, dtype=np.float64)
    wall, idle, steps = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    _check(lib().smpu_sched_simulate(_p(t), t.size, workers, update_freq, ctypes.byref(wall), ctypes.byref(idle),
                                     ctypes.byref(steps)), "simulate")
    return dict(wall=wall.value, idle_fraction=idle.value, steps=steps.value)


def overlap_schedule(layer_bytes, backward_seconds, threshold_bytes, latency_seconds, bytes_per_second, workers):
    """SPEC S:405-413 (include/smpu_sched.h): -> dict(buckets=[(last_layer, ready, start, end)], total_overlap,
    total_serial)."""
    b = np.ascontiguousarray(layer_bytes, dtype=np.float64)
    t = np.ascontiguousarray(backward_seconds, dtype=np.float64)
    cap = max(b.size, 1)
    last = np.zeros(cap, np.int64)
    ready, start, end = (np.zeros(cap, np.float64) for _ in range(3))
    nb, tov, tser = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    _check(lib().smpu_sched_overlap_schedule(_p(b), _p(t), b.size, float(threshold_bytes), float(latency_seconds),
                                             float(bytes_per_second), int(workers), _p(last), _p(ready), _p(start),
                                             _p(end), cap, ctypes.byref(nb), ctypes.byref(tov), ctypes.byref(tser)),
           "overlap_schedule")
    k = nb.value
    return dict(buckets=[(int(last[i]), ready[i], start[i], end[i]) for i in range(k)], total_overlap=tov.value,
                total_serial=tser.value)
