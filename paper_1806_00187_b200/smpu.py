"""Thin ctypes binding of libsmpu.so (include/smpu.h): argument marshalling only.

Every step of the update runs in the library's sm_100a kernels; there is no
Python or CPU fallback.  If the library is missing the import fails loudly.
Functions keep the C names without the `smpu_` prefix; `UpdateStep` wraps a ctx.
torch tensors are accepted wherever the C ABI takes a pointer (their data_ptr is
passed); numpy arrays are passed as host pointers.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsmpu.so")

OK, EINVAL, ESTATE, ECUDA, ENCCL, ENOMEM, EPOISONED = range(7)
STATE_MASTER, STATE_M, STATE_V, STATE_W16, STATE_ACCUM, STATE_SCALARS = range(6)
K1_FIRST, K1_ADD, K1S, K0, K2, KCAST, ALLREDUCE, DECISION_AR, K1_MANY, K12, N_KERNELS = range(11)
KERNEL_NAMES = ["k1_first", "k1_add", "k1s_sweep", "k0_decide", "k2_adam", "kc_cast", "allreduce", "decision_ar",
                "k1_many", "k12_fused"]
GRAPH_STREAMING, GRAPH_RESIDENT = 0, 1
STREAM_NAMES = ["caller", "allreduce", "decision", "adam_per_bucket"]
AR_AUTO, AR_NCCL, AR_FUSED = range(3)
NCCL_ID_BYTES = 128


class SmpuError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"smpu status {status}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("peak_lr", ctypes.c_double), ("warmup_updates", ctypes.c_int64), ("beta1", ctypes.c_double),
                ("beta2", ctypes.c_double), ("eps", ctypes.c_double), ("init_scale_log2", ctypes.c_int32),
                ("min_scale_log2", ctypes.c_int32), ("max_scale_log2", ctypes.c_int32),
                ("growth_interval", ctypes.c_int64), ("update_freq", ctypes.c_int32),
                ("bucket_bytes", ctypes.c_int64), ("allreduce", ctypes.c_int32), ("sharded", ctypes.c_int32),
                ("fuse_final", ctypes.c_int32), ("accum_fp32", ctypes.c_int32), ("split_tensors", ctypes.c_int32),
                ("ar_ctas", ctypes.c_int32), ("ar_threads", ctypes.c_int32), ("ar_vec_bytes", ctypes.c_int32),
                ("ar_unroll", ctypes.c_int32), ("ar_mcast", ctypes.c_int32), ("pdl", ctypes.c_int32),
                ("ar_pieces", ctypes.c_int32), ("ar_copy_engine", ctypes.c_int32)]


class StepResult(ctypes.Structure):
    _fields_ = [("overflow", ctypes.c_int32), ("applied", ctypes.c_int32), ("scale_log2_used", ctypes.c_int32),
                ("scale_log2_next", ctypes.c_int32), ("lr", ctypes.c_float), ("discarded", ctypes.c_int32),
                ("num_updates", ctypes.c_int64), ("ntokens_total", ctypes.c_int64), ("clean_streak", ctypes.c_int64),
                ("attempt", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["smpu_abi_version", "smpu_config_default", "smpu_unique_id", "smpu_plan_buckets", "smpu_init",
           "smpu_group_init", "smpu_group_member", "smpu_group_destroy",
           "smpu_num_params", "smpu_accumulator", "smpu_shard_ranges", "smpu_plan_shards", "smpu_allreduce_impl", "smpu_buckets",
           "smpu_weights_fp16", "smpu_loss_scale", "smpu_accumulate", "smpu_accumulate_many", "smpu_micro_begin",
           "smpu_accumulate_bucket", "smpu_tensor_ready", "smpu_step", "smpu_allreduce_accumulator", "smpu_graph_capture",
           "smpu_graph_launch", "smpu_result", "smpu_get_master", "smpu_get_state", "smpu_set_state",
           "smpu_set_timing", "smpu_kernel_stats", "smpu_kernel_trace", "smpu_last_error", "smpu_destroy"]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        p, i64, i32, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int
        P = ctypes.POINTER
        sig = {
            "smpu_abi_version": ([], i32),
            "smpu_config_default": ([P(Config)], st),
            "smpu_unique_id": ([p, i64], st),
            "smpu_plan_buckets": ([p, i32, i64, P(ctypes.c_int), p], st),
            "smpu_init": ([P(p), P(Config), i32, i32, p, i32, p, i32, p], st),
            "smpu_group_init": ([P(p), P(Config), i32, i32, p, i32, p], st),
            "smpu_group_member": ([p, i32, P(p)], st),
            "smpu_group_destroy": ([p], None),
            "smpu_num_params": ([p, P(ctypes.c_int64)], st),
            "smpu_allreduce_impl": ([p, P(ctypes.c_int)], st),
            "smpu_shard_ranges": ([p, p, i32, P(ctypes.c_int)], st),
            "smpu_plan_shards": ([p, i32, i32, i32, p, i32, P(ctypes.c_int)], st),
            "smpu_buckets": ([p, P(ctypes.c_int), p], st),
            "smpu_weights_fp16": ([p, P(p)], st),
            "smpu_accumulator": ([p, P(p)], st),
            "smpu_loss_scale": ([p, P(p)], st),
            "smpu_accumulate": ([p, p, i64, p], st),
            "smpu_micro_begin": ([p, i64], st),
            "smpu_accumulate_many": ([p, p, p, i32, p], st),
            "smpu_accumulate_bucket": ([p, i32, p, p], st),
            "smpu_tensor_ready": ([p, i32, p], st),
            "smpu_step": ([p, p, P(StepResult)], st),
            "smpu_result": ([p, i64, P(StepResult)], st),
            "smpu_allreduce_accumulator": ([p, p], st),
            "smpu_graph_capture": ([p, p, i32, i32], st),
            "smpu_graph_launch": ([p, p, i32, p], st),
            "smpu_get_master": ([p, p, i64], st),
            "smpu_get_state": ([p, i32, p, i64], st),
            "smpu_set_state": ([p, i32, p, i64], st),
            "smpu_set_timing": ([p, i32], st),
            "smpu_kernel_stats": ([p, p, p, i32], st),
            "smpu_kernel_trace": ([p, p, p, p, p, i64, P(ctypes.c_int64)], st),
            "smpu_last_error": ([], ctypes.c_char_p),
            "smpu_destroy": ([p], None),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def last_error() -> str:
    return lib().smpu_last_error().decode()


def _check(status):
    if status != OK:
        raise SmpuError(status, last_error())


def _ptr(x):
    """torch tensor -> data_ptr; numpy array -> host pointer; int -> as is; None -> NULL."""
    if x is None:
        return None
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    raise TypeError(type(x))


def _stream(s, device: int):
    if s is None:                  # torch's current stream on the ctx's device (not on torch's current device)
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    if isinstance(s, int):
        return ctypes.c_void_p(s)
    return ctypes.c_void_p(s.cuda_stream)


def abi_version() -> int:
    return lib().smpu_abi_version()


def config_default(**kw) -> Config:
    c = Config()
    _check(lib().smpu_config_default(ctypes.byref(c)))
    for k, v in kw.items():
        if not hasattr(c, k):
            raise AttributeError(k)
        setattr(c, k, v)
    return c


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(lib().smpu_unique_id(buf, NCCL_ID_BYTES))
    return buf.raw


def plan_buckets(numel, bucket_bytes: int) -> np.ndarray:
    numel = np.ascontiguousarray(numel, dtype=np.int64)
    nb = ctypes.c_int()
    out = np.zeros(numel.size + 1, dtype=np.int64)
    _check(lib().smpu_plan_buckets(_ptr(numel), numel.size, bucket_bytes, ctypes.byref(nb), _ptr(out)))
    return out[: nb.value + 1].copy()


def plan_shards(bucket_begin, world: int, rank: int):
    """Host-only: [(lo, hi)] element ranges rank `rank` of `world` updates in the sharded layout."""
    bb = np.ascontiguousarray(bucket_begin, dtype=np.int64)
    cnt = ctypes.c_int()
    _check(lib().smpu_plan_shards(_ptr(bb), bb.size - 1, world, rank, None, 0, ctypes.byref(cnt)))
    buf = np.zeros(2 * max(cnt.value, 1), dtype=np.int64)
    _check(lib().smpu_plan_shards(_ptr(bb), bb.size - 1, world, rank, _ptr(buf), cnt.value, ctypes.byref(cnt)))
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt.value)]


class UpdateStep:
    """One library ctx: init(world, buckets, params) / accumulate(micro_grads, ntokens) / step() / get_master()."""

    def __init__(self, numel, init_params, cfg: Config | None = None, world: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, device: int = 0, _member=None):
        self.cfg = cfg or config_default()
        self._owned = _member is None
        if _member is not None:          # a member of a VirtualGroup (the group owns the ctx)
            self._ctx = _member
        else:
            numel = np.ascontiguousarray(numel, dtype=np.int64)
            self._ctx = ctypes.c_void_p()
            idbuf = ctypes.create_string_buffer(nccl_id, NCCL_ID_BYTES) if nccl_id is not None else None
            _check(lib().smpu_init(ctypes.byref(self._ctx), ctypes.byref(self.cfg), world, rank, idbuf, device,
                                   _ptr(numel), numel.size, _ptr(init_params)))
        n = ctypes.c_int64()
        _check(lib().smpu_num_params(self._ctx, ctypes.byref(n)))
        self.n = n.value
        nb = ctypes.c_int()
        _check(lib().smpu_buckets(self._ctx, ctypes.byref(nb), None))
        self.bucket_begin = np.zeros(nb.value + 1, dtype=np.int64)
        _check(lib().smpu_buckets(self._ctx, ctypes.byref(nb), _ptr(self.bucket_begin)))
        self.world, self.rank, self.device = world, rank, device

    # -------------------------------------------------------------- hot path
    def accumulate(self, micro_grads, ntokens: int, stream=None):
        _check(lib().smpu_accumulate(self._ctx, _ptr(micro_grads), int(ntokens), _stream(stream, self.device)))

    def micro_begin(self, ntokens: int):
        _check(lib().smpu_micro_begin(self._ctx, int(ntokens)))

    def accumulate_bucket(self, bucket: int, bucket_grads, stream=None):
        _check(lib().smpu_accumulate_bucket(self._ctx, bucket, _ptr(bucket_grads), _stream(stream, self.device)))

    def tensor_ready(self, tensor: int, stream=None):
        _check(lib().smpu_tensor_ready(self._ctx, tensor, _stream(stream, self.device)))

    def step(self, stream=None, wait: bool = True):
        """wait=True: returns the result dict; wait=False: asynchronous, returns None."""
        if not wait:
            _check(lib().smpu_step(self._ctx, _stream(stream, self.device), None))
            return None
        r = StepResult()
        _check(lib().smpu_step(self._ctx, _stream(stream, self.device), ctypes.byref(r)))
        return r.as_dict()

    def accumulate_many(self, micro_grads, ntokens, stream=None):
        arr = (ctypes.c_void_p * len(micro_grads))(*[_ptr(g).value for g in micro_grads])
        toks = np.ascontiguousarray(ntokens, dtype=np.int64)
        _check(lib().smpu_accumulate_many(self._ctx, arr, _ptr(toks), len(micro_grads), _stream(stream, self.device)))

    def graph_capture(self, micro_grads, resident: bool = False):
        """Record update_freq x accumulate(micro_grads[k]) + step as one CUDA graph (device buffers);
        resident=True records one accumulate_many over all of them instead."""
        arr = (ctypes.c_void_p * len(micro_grads))(*[_ptr(g).value for g in micro_grads])
        _check(lib().smpu_graph_capture(self._ctx, arr, len(micro_grads), GRAPH_RESIDENT if resident else 0))

    def graph_launch(self, ntokens, stream=None):
        toks = np.ascontiguousarray(ntokens, dtype=np.int64)
        _check(lib().smpu_graph_launch(self._ctx, _ptr(toks), toks.size, _stream(stream, self.device)))

    def allreduce_accumulator(self, stream=None):
        _check(lib().smpu_allreduce_accumulator(self._ctx, _stream(stream, self.device)))

    def result(self, attempt: int):
        r = StepResult()
        _check(lib().smpu_result(self._ctx, attempt, ctypes.byref(r)))
        return r.as_dict()

    # -------------------------------------------------------------- accessors
    def shard_ranges(self):
        """[(lo, hi)] element ranges whose theta/m/v this rank updates (everything unless sharded)."""
        cnt = ctypes.c_int()
        _check(lib().smpu_shard_ranges(self._ctx, None, 0, ctypes.byref(cnt)))
        buf = np.zeros(2 * max(cnt.value, 1), dtype=np.int64)
        _check(lib().smpu_shard_ranges(self._ctx, _ptr(buf), cnt.value, ctypes.byref(cnt)))
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt.value)]

    @property
    def allreduce_impl(self) -> int:
        v = ctypes.c_int()
        _check(lib().smpu_allreduce_impl(self._ctx, ctypes.byref(v)))
        return v.value

    @property
    def n_buckets(self):
        return len(self.bucket_begin) - 1

    def weights_fp16_ptr(self) -> int:
        p = ctypes.c_void_p()
        _check(lib().smpu_weights_fp16(self._ctx, ctypes.byref(p)))
        return p.value

    def accumulator_ptr(self) -> int:
        """Device pointer of the fp16[n] accumulator, for producers that accumulate in place (then pass
        micro_grads=None to accumulate / accumulate_bucket)."""
        p = ctypes.c_void_p()
        _check(lib().smpu_accumulator(self._ctx, ctypes.byref(p)))
        return p.value

    def loss_scale_ptr(self) -> int:
        p = ctypes.c_void_p()
        _check(lib().smpu_loss_scale(self._ctx, ctypes.byref(p)))
        return p.value

    def get_master(self, out=None):
        out = np.empty(self.n, dtype=np.float32) if out is None else out
        _check(lib().smpu_get_master(self._ctx, _ptr(out), self.n))
        return out

    _STATE_DTYPES = {STATE_MASTER: np.float32, STATE_M: np.float32, STATE_V: np.float32, STATE_W16: np.uint16,
                     STATE_ACCUM: np.uint16}

    def get_state(self, which: int, out=None):
        if which == STATE_SCALARS:
            out = np.empty(4, dtype=np.int64) if out is None else out
            _check(lib().smpu_get_state(self._ctx, which, _ptr(out), 32))
            return out
        out = np.empty(self.n, dtype=self._STATE_DTYPES[which]) if out is None else out
        nbytes = out.numel() * out.element_size() if hasattr(out, "element_size") else out.nbytes
        _check(lib().smpu_get_state(self._ctx, which, _ptr(out), nbytes))
        return out

    def set_state(self, which: int, src):
        nbytes = src.numel() * src.element_size() if hasattr(src, "element_size") else src.nbytes
        _check(lib().smpu_set_state(self._ctx, which, _ptr(src), nbytes))

    def scalars(self):
        e, clean, t, attempts = self.get_state(STATE_SCALARS)
        return dict(e=int(e), clean=int(clean), t=int(t), attempts=int(attempts))

    def set_timing(self, enable: bool):
        _check(lib().smpu_set_timing(self._ctx, int(enable)))

    def kernel_stats(self, reset: bool = False):
        launches = np.zeros(N_KERNELS, dtype=np.int64)
        ms = np.zeros(N_KERNELS, dtype=np.float64)
        _check(lib().smpu_kernel_stats(self._ctx, _ptr(launches), _ptr(ms), int(reset)))
        return {KERNEL_NAMES[k]: dict(launches=int(launches[k]), ms=float(ms[k])) for k in range(N_KERNELS)}

    def kernel_trace(self):
        """[(kernel, stream, start_ms, end_ms)] of the launches timed since the last stats reset."""
        cnt = ctypes.c_int64()
        _check(lib().smpu_kernel_trace(self._ctx, None, None, None, None, 0, ctypes.byref(cnt)))
        m = cnt.value
        kind = np.zeros(m, np.int32)
        strm = np.zeros(m, np.int32)
        t0 = np.zeros(m, np.float64)
        t1 = np.zeros(m, np.float64)
        _check(lib().smpu_kernel_trace(self._ctx, _ptr(kind), _ptr(strm), _ptr(t0), _ptr(t1), m, ctypes.byref(cnt)))
        return [(KERNEL_NAMES[k], STREAM_NAMES[s], a, b) for k, s, a, b in zip(kind, strm, t0, t1)]

    def close(self):
        if self._ctx:
            if self._owned:
                lib().smpu_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class VirtualGroup:
    """smpu_group_init: `world` data-parallel ranks held on one GPU (the world > 1 kernels over local windows).
    `members[r]` is rank r's UpdateStep; drive them like W processes would (include/smpu.h states the two rules)."""

    def __init__(self, numel, init_params, cfg: Config | None = None, world: int = 2, device: int = 0):
        self.cfg = cfg or config_default()
        numel = np.ascontiguousarray(numel, dtype=np.int64)
        self._g = ctypes.c_void_p()
        _check(lib().smpu_group_init(ctypes.byref(self._g), ctypes.byref(self.cfg), world, device, _ptr(numel),
                                     numel.size, _ptr(init_params)))
        self.world = world
        self.members = []
        for r in range(world):
            m = ctypes.c_void_p()
            _check(lib().smpu_group_member(self._g, r, ctypes.byref(m)))
            self.members.append(UpdateStep(numel, None, self.cfg, world=world, rank=r, device=device, _member=m))

    def close(self):
        if self._g:
            for m in self.members:
                m.close()
            lib().smpu_group_destroy(self._g)
            self._g = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
