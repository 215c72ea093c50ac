"""Seeded synthetic input generators (shared by tests, smoke and bench).

Holds none of the method's arithmetic; see synth.c for the recipe.  CPU side
(libsynth.so) feeds the oracle; GPU side (libsynth_gpu.so) fills device
buffers for the CUDA path at full size.  Injection overrides (the fault
injector of SURVEY.md 8(d.2)) are applied here, identically for both sides.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .models import WORKLOADS, Workload, base_ende, big_ende, big_enfr, tiny, transformer_tensors  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
FAMILIES = {"real": 0, "exact": 1, "zero": 2}
INF16, NINF16, NAN16, MAX16, R40000, R20000 = 0x7C00, 0xFC00, 0x7E00, 0x7BFF, 0x78E2, 0x74E2

_lib = None
_glib = None


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        u64, i64, i32, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.synth_mix.restype = u64
        lib.synth_mix.argtypes = [u64]
        lib.synth_key.restype = u64
        lib.synth_key.argtypes = [u64, u64, u64, u64]
        lib.synth_ntokens.restype = i64
        lib.synth_ntokens.argtypes = [u64]
        lib.synth_fill.argtypes = [p, i32, p, p, i32, u64, i32, i32]
        lib.synth_fill_range.argtypes = [p, i64, i64, i32, p, p, i32, u64, i32, i32]
        lib.synth_sample.argtypes = [p, p, i64, i32, p, p, i32, u64, i32, i32]
        lib.synth_theta0.argtypes = [p, i64, u64]
        lib.synth_theta0_sample.argtypes = [p, p, i64, u64]
        lib.synth_embed_rows.restype = i64
        lib.synth_embed_rows.argtypes = [p, i64, u64, i64, ctypes.c_double]
        _lib = lib
    return _lib


def _load_gpu():
    global _glib
    if _glib is None:
        path = os.path.join(_HERE, "libsynth_gpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        u64, i64, i32, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.synth_gpu_fill.restype = i32
        lib.synth_gpu_fill.argtypes = [p, i32, p, p, i32, u64, i32, i32, p]
        lib.synth_gpu_fill_all.restype = i32
        lib.synth_gpu_fill_all.argtypes = [p, i64, p, p, i32, i32, u64, i32, i32, p]
        lib.synth_gpu_theta0.restype = i32
        lib.synth_gpu_theta0.argtypes = [p, i64, u64, p]
        _glib = lib
    return _glib


def mix(x: int) -> int:
    return _load().synth_mix(x & 0xFFFFFFFFFFFFFFFF)


def key(seed: int, u: int, r: int, k: int) -> int:
    return _load().synth_key(seed, u, r, k)


def ntokens(wl: Workload, u: int, r: int, k: int) -> int:
    return _load().synth_ntokens(key(wl.seed, u, r, k))


def theta0_key(wl: Workload) -> int:
    return key(wl.seed, 0, 0xFFFF, 0)


def exact_K(world: int, update_freq: int) -> int:
    return 2048 // (world * update_freq)


class Layout:
    """Packed offsets of a workload's tensors (ready order, no padding)."""

    def __init__(self, wl: Workload):
        self.begin = np.zeros(len(wl.tensors) + 1, dtype=np.int64)
        self.begin[1:] = np.cumsum(np.asarray(wl.numel, dtype=np.int64))
        self.cls = np.asarray(wl.classes, dtype=np.int32)
        self.n = int(self.begin[-1])
        self.n_tensors = len(wl.tensors)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def overrides(wl: Workload, u: int, r: int, k: int):
    """Injected (index, fp16 bits) for micro-gradient (u, r, k); k is 1-based.

    INF/NINF/NAN write the pattern at (u, r, k, i).  ACC_OVF: 65504 at k=1,2 on rank r,
    every other contribution at i zero (overflow by local accumulation).  RED_OVF:
    40000 at k=c on every rank, every other contribution at i zero (overflow only after
    the cross-rank sum; needs W >= 2).  BIG: 20000 at k=c on ranks 0 and 1, every other contribution at i
    zero (a finite 40000 after the sum, large enough that the early decision of the W > 1 path must defer
    to the sweep of R)."""
    out = []
    c, W = wl.update_freq, wl.world
    for inj in wl.injections:
        if inj["u"] != u:
            continue
        kind, i = inj["kind"], inj["i"]
        if kind in ("INF", "NINF", "NAN"):
            if r == inj["r"] and k == inj["k"]:
                out.append((i, {"INF": INF16, "NINF": NINF16, "NAN": NAN16}[kind]))
        elif kind == "ACC_OVF":
            if c < 2:
                raise ValueError("ACC_OVF needs update_freq >= 2")
            out.append((i, MAX16 if (r == inj["r"] and k in (1, 2)) else 0))
        elif kind == "RED_OVF":
            if W < 2:
                raise ValueError("RED_OVF needs world >= 2")
            out.append((i, R40000 if k == c else 0))
        elif kind == "BIG":
            if W < 2:
                raise ValueError("BIG needs world >= 2")
            out.append((i, R20000 if (k == c and r < 2) else 0))
        else:
            raise ValueError(kind)
    return out


ZIPF_S = 1.1   # token ids ~ Zipf(1.1)


def embed_mask(wl: Workload, n_rows: int, u: int, r: int, k: int) -> np.ndarray:
    """Rows of an embedding tensor that carry gradient in micro-batch (u, r, k): those of its ntokens(u, r, k) token
    ids, drawn from Zipf(1.1) over the rows (synth_embed_rows).  uint8[n_rows]; one array for both fills."""
    mask = np.empty(n_rows, dtype=np.uint8)
    kk = key(wl.seed, u, r, k)
    if _load().synth_embed_rows(_ptr(mask), n_rows, kk, _load().synth_ntokens(kk), ZIPF_S) < 0:
        raise MemoryError("synth_embed_rows")
    return mask


def embed_spans(wl: Workload, lay: Layout):
    """[(lo, hi, n_rows)] of the embedding tensors when the workload's embedding gradient is row-sparse."""
    if not wl.embed_row:
        return []
    return [(int(lay.begin[j]), int(lay.begin[j + 1]), -(-int(lay.begin[j + 1] - lay.begin[j]) // wl.embed_row))
            for j in range(lay.n_tensors) if lay.cls[j] == 2]


def _apply_rows_range(out, lo, hi, wl, lay, u, r, k):
    """Zero out[i - lo] for i in [lo, hi) in an embedding row that holds no token of the micro-batch."""
    for a, b, rows in embed_spans(wl, lay):
        s0, s1 = max(a, lo), min(b, hi)
        if s0 >= s1:
            continue
        mask = embed_mask(wl, rows, u, r, k)
        keep = mask[(np.arange(s0, s1) - a) // wl.embed_row].astype(bool)
        out[s0 - lo:s1 - lo][~keep] = 0


def micro_grad_cpu(wl: Workload, lay: Layout, u: int, r: int, k: int, e: int, family: str | None = None):
    """Full packed fp16 micro-gradient g_{r,k} of update u (uint16 bit patterns)."""
    fam = FAMILIES[family or wl.family]
    out = np.empty(lay.n, dtype=np.uint16)
    _load().synth_fill(_ptr(out), lay.n_tensors, _ptr(lay.begin), _ptr(lay.cls), fam,
                       key(wl.seed, u, r, k), e, exact_K(wl.world, wl.update_freq))
    _apply_rows_range(out, 0, lay.n, wl, lay, u, r, k)
    for i, bits in overrides(wl, u, r, k):
        out[i] = bits
    return out


def micro_grad_range(wl: Workload, lay: Layout, lo: int, hi: int, u: int, r: int, k: int, e: int,
                     family: str | None = None):
    """g_{r,k}[lo:hi] (uint16 bit patterns), injections included."""
    fam = FAMILIES[family or wl.family]
    out = np.empty(hi - lo, dtype=np.uint16)
    _load().synth_fill_range(_ptr(out), lo, hi, lay.n_tensors, _ptr(lay.begin), _ptr(lay.cls), fam,
                             key(wl.seed, u, r, k), e, exact_K(wl.world, wl.update_freq))
    _apply_rows_range(out, lo, hi, wl, lay, u, r, k)
    for i, bits in overrides(wl, u, r, k):
        if lo <= i < hi:
            out[i - lo] = bits
    return out


def micro_grad_sample(wl: Workload, lay: Layout, idx: np.ndarray, u: int, r: int, k: int, e: int,
                      family: str | None = None):
    """g_{r,k}[idx] computed one by one (for sampled parity at full size)."""
    fam = FAMILIES[family or wl.family]
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.size, dtype=np.uint16)
    _load().synth_sample(_ptr(out), _ptr(idx), idx.size, lay.n_tensors, _ptr(lay.begin), _ptr(lay.cls), fam,
                         key(wl.seed, u, r, k), e, exact_K(wl.world, wl.update_freq))
    for a, b, rows in embed_spans(wl, lay):
        sel = (idx >= a) & (idx < b)
        if sel.any():
            mask = embed_mask(wl, rows, u, r, k)
            out[sel] = np.where(mask[(idx[sel] - a) // wl.embed_row].astype(bool), out[sel], 0)
    ov = overrides(wl, u, r, k)
    if ov:
        pos = {int(v): j for j, v in enumerate(idx)}
        for i, bits in ov:
            if i in pos:
                out[pos[i]] = bits
    return out


def theta0_cpu(wl: Workload, lay: Layout):
    out = np.empty(lay.n, dtype=np.float32)
    _load().synth_theta0(_ptr(out), lay.n, theta0_key(wl))
    return out


def theta0_sample(wl: Workload, idx: np.ndarray):
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.size, dtype=np.float32)
    _load().synth_theta0_sample(_ptr(out), _ptr(idx), idx.size, theta0_key(wl))
    return out


# ---------------------------------------------------------------- GPU side (torch tensors)
def micro_grad_gpu(out, wl: Workload, lay: Layout, u: int, r: int, k: int, e: int, family: str | None = None,
                   stream=None):
    """Fill a device int16/uint16/float16 torch tensor of lay.n elements with g_{r,k}."""
    import torch
    fam = FAMILIES[family or wl.family]
    s = stream if stream is not None else torch.cuda.current_stream()
    dev = getattr(lay, "_dev_table", None)
    if dev is None or dev[0].device != out.device:
        dev = (torch.from_numpy(lay.begin).to(out.device), torch.from_numpy(lay.cls).to(out.device))
        lay._dev_table = dev
    rc = _load_gpu().synth_gpu_fill_all(ctypes.c_void_p(out.data_ptr()), lay.n, ctypes.c_void_p(dev[0].data_ptr()),
                                        ctypes.c_void_p(dev[1].data_ptr()), lay.n_tensors, fam,
                                        key(wl.seed, u, r, k), e, exact_K(wl.world, wl.update_freq),
                                        ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_gpu_fill: cuda error {rc}")
    for a, b, rows in embed_spans(wl, lay):     # the same mask array as the CPU fill (embed_mask)
        with torch.cuda.stream(s):
            mask = torch.from_numpy(embed_mask(wl, rows, u, r, k).astype(bool)).to(out.device)
            seg = out.view(torch.int16)[a:b]
            full = (b - a) // wl.embed_row
            if full:
                seg[:full * wl.embed_row].view(full, wl.embed_row)[~mask[:full]] = 0
            if full < rows and not bool(mask[rows - 1]):
                seg[full * wl.embed_row:] = 0
    ov = overrides(wl, u, r, k)
    if ov:
        with torch.cuda.stream(s):
            flat = out.view(torch.int16)
            idx = torch.tensor([i for i, _ in ov], dtype=torch.int64, device=out.device)
            val = torch.tensor(np.asarray([b for _, b in ov], dtype=np.uint16).view(np.int16), device=out.device)
            flat[idx] = val
    return out


def theta0_gpu(out, wl: Workload, stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _load_gpu().synth_gpu_theta0(ctypes.c_void_p(out.data_ptr()), out.numel(), theta0_key(wl),
                                      ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_gpu_theta0: cuda error {rc}")
    return out
