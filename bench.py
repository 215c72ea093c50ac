#!/usr/bin/env python
"""Benchmark of the synchronous mixed-precision large-batch update step (arXiv 1806.00187 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config big_ende|base|tiny] [--impl ours|reference]

One step = one whole update: update_freq x accumulate (K1) + bucketed all-reduce (W > 1) + step (decision + Adam),
on synthetic Transformer-shaped fp16 micro-gradients already resident in HBM.  N > 1: one process per GPU, launched
by torchrun or, without it, by bench.py itself; rank 0 prints ONE JSON line.  At W > 1 the headline is the paper's
replicated update, with the sharded variant (f2) beside it.  Metric and config: BASELINE.json
(configs[2], Transformer-big En-De, update_freq 16, at 1/2/4/8 B200).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "update steps/s & grad elems/s at 1/2/4/8 B200; HBM GB/s and bus GB/s vs peak"
UNIT = "grad elems/s"
NVLINK_NOMINAL_GBS = 900.0
# measured NVLink roofline of the all-reduce's traffic shape on this pool: SM 256-bit loads from and stores to a peer
# at once, per direction (tools/nvlink_probe.cu "pullpush", best shape, 4 x B200: profiles/r2/j_w4/nvlink_probe.jsonl)
NVLINK_MEASURED_GBS = 675.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="big_ende", choices=["big_ende", "base", "tiny", "big_enfr"])
    ap.add_argument("--update-freq", type=int, default=None)
    ap.add_argument("--bucket-mib", type=float, default=150.0)
    ap.add_argument("--allreduce", choices=["auto", "nccl", "fused"], default="auto")
    ap.add_argument("--optimizer", choices=["auto", "sharded", "replicated"], default="auto",
                    help="W > 1 update layout of the headline. replicated = every rank updates the whole vector (the "
                         "paper's layout, SURVEY 8(e)); sharded = SURVEY f2: reduce-scatter + Adam on 1/W + "
                         "all-gather of w16 (bitwise equal to the replicated update); auto = replicated headline "
                         "with the sharded variant timed beside it when the fused all-reduce is available")
    ap.add_argument("--sharded", action="store_true", help="same as --optimizer sharded")
    ap.add_argument("--ar-pieces", type=int, default=None,
                    help="smpu_config.ar_pieces (replicated, W > 1): every bucket's all-reduce in pieces, "
                         "each followed by its Adam; default 2 (measured best or equal at W = 2 / 4, c = 16 / 1: "
                         "profiles/r2/f_w4/c4_w4_pieces.jsonl)")
    ap.add_argument("--ar-ctas", type=int, default=0, help="smpu_config.ar_ctas (0: one per SM)")
    ap.add_argument("--ar-unroll", type=int, choices=[1, 2], default=1, help="smpu_config.ar_unroll")
    ap.add_argument("--ar-threads", type=int, choices=[256, 512], default=256, help="smpu_config.ar_threads")
    ap.add_argument("--ar-copy-engine", type=int, choices=[0, 1, 2], default=None,
                    help="smpu_config.ar_copy_engine (replicated, W > 1): the bucket all-reduce's NVLink traffic by "
                         "the copy engines (cudaMemcpyAsync push + all-gather, SM fold only); 2: all buckets but the "
                         "last.  Default: 0 in m1 (the HBM-bound update step alone: the SM kernel moves the fewest "
                         "HBM bytes), 1 in m2 / train (a backward runs beside the exchange: keep its SMs)")
    ap.add_argument("--generator", choices=["real", "exact", "zero", "real_sparse"], default="real",
                    help="input family (SURVEY 8(d.2)); real_sparse = G_real with the row-sparse embedding gradient "
                         "(Zipf(1.1) token rows); the performance-independence check times all four")
    ap.add_argument("--accum-fp32", action="store_true",
                    help="SURVEY Z1 knob (smpu_config.accum_fp32): fp32 accumulator, rn16 of the last sum")
    ap.add_argument("--fuse-final", type=int, choices=[0, 1], default=0,
                    help="W = 1 headline: 0 (the library default, SURVEY 8(b)'s contract) = accumulate, decide, then "
                         "Adam; 1 = the opt-in smpu_config.fuse_final (last micro-batch fused into Adam).  With 0 the "
                         "fused variant is timed beside the headline")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the call-by-call path (c x smpu_accumulate + smpu_step) instead of the captured "
                         "CUDA graph of the same update (smpu_graph_capture / smpu_graph_launch)")
    ap.add_argument("--m2-fused", action="store_true",
                    help="M2 with SURVEY f3's producer: dW GEMMs accumulate in place into smpu_accumulator "
                         "(cuBLAS beta = 1; bitwise the paper's accumulate), 1-D tensors by fp16 add, no K1")
    ap.add_argument("--trace", default=None, help="write the timed launches (per stream) as JSONL here")
    ap.add_argument("--mode", choices=["m1", "m2", "train"], default="m1",
                    help="m1: the update step alone (headline); m2: with a cuBLAS backward-load emulator so the "
                         "bucket all-reduces overlap backward as in the paper's Fig. 3 (exposed-comm measurement); "
                         "train: the real Transformer-big forward + backward (producer/transformer.py) feeding the "
                         "library, buckets handed over as backward finishes them (SURVEY f3; Table 1-style tok/s)")
    ap.add_argument("--tokens", type=int, default=3500, help="train: token budget per micro-batch (P:317)")
    ap.add_argument("--sent-len", type=int, default=28, help="train: sentence length of the synthetic batches")
    ap.add_argument("--eager-producer", action="store_true",
                    help="train: run the producer eagerly (Python-launch bound) instead of as a CUDA graph per shape")
    ap.add_argument("--no-overlap", action="store_true",
                    help="train: hand the last micro-batch over after backward (no overlap) instead of per bucket")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle cpu_baseline leg")
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: oracle seconds for the whole run, spread over the steps")
    args = ap.parse_args()
    if args.ar_copy_engine is None:
        args.ar_copy_engine = 0 if args.mode == "m1" else 1
    if args.ar_pieces is None:
        args.ar_pieces = 2 if args.gpus > 1 else 1
    return args


def set_generator(wl, generator):
    """--generator: the input family, and for real_sparse the row-sparse embedding (rows of d elements)."""
    wl.family = "real" if generator == "real_sparse" else generator
    if generator == "real_sparse":
        wl.embed_row = {"transformer_big_ende": 1024, "transformer_big_enfr": 1024, "transformer_base_ende": 512}.get(wl.name, 64)
    return wl


def workload(name, world, update_freq):
    from synth import models
    if name == "big_ende":
        return models.big_ende(world, update_freq or 16)
    if name == "base":
        return models.base_ende(world, update_freq or 1)
    if name == "big_enfr":
        wl = models.big_enfr(world, update_freq or 16)
        wl.injections, wl.family = [], "real"
        return wl
    wl = models.tiny()
    wl.injections = []
    wl.world = world
    if update_freq:
        wl.update_freq = update_freq
    return wl


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 6:
                    try:
                        rows.append((float(parts[0]), float(parts[1]), parts[2:]))
                    except ValueError:
                        pass
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for _, _, fl in rows for j, v in enumerate(fl) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------------ oracle legs
def oracle_rate(wl, seconds, slice_elems=2_000_000):
    """The oracle as it stands on a bounded sample: full update steps (all c micro-batches, W ranks emulated)
    over a contiguous slice of the parameter vector; returns grad elems/s and the sample description."""
    import oracle as O
    import synth
    lay = synth.Layout(wl)
    lo = 0
    hi = min(lay.n, slice_elems)
    W, c = wl.world, wl.update_freq
    theta0 = synth.theta0_cpu(wl, lay)[lo:hi] if lay.n <= 4 * slice_elems else \
        synth.theta0_sample(wl, np.arange(lo, hi, dtype=np.int64))
    orc = O.Oracle(theta0)
    grads = [[synth.micro_grad_range(wl, lay, lo, hi, 1, r, k, orc.e) for k in range(1, c + 1)] for r in range(W)]
    toks = [[synth.ntokens(wl, 1, r, k) for k in range(1, c + 1)] for r in range(W)]
    t0 = time.perf_counter()
    n_up = 0
    while True:                        # seconds = 0: exactly one whole update of the slice
        orc.update(grads, toks)
        n_up += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    value = W * c * (hi - lo) * n_up / dt
    sample = (f"{n_up} oracle update(s) of elements [{lo}, {hi}) of {wl.name} (W={W} ranks emulated, "
              f"c={c}), {dt:.1f} s")
    return value, dt / n_up, sample


def omp_threads():
    """The oracle's OpenMP thread count in effect (what `cores` reports)."""
    import oracle as O
    return O.set_threads(0)


def cpu_model():
    """Host CPU model (lscpu 'Model name'), for the oracle baselines."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def plan_buckets_host(numel, bucket_bytes):
    """The paper's bucket rule (reading R17) restated for the reference arm's config description only: greedy
    in ready order, whole tensors, close at >= threshold, remainder last.  (The product's plan is smpu_plan_buckets.)"""
    n_b, cur = 0, 0
    for x in numel:
        cur += 2 * int(x)
        if cur >= bucket_bytes:
            n_b, cur = n_b + 1, 0
    return n_b + (1 if cur else 0)


def bench_config(args, wl, world, toks_per_update, path_bytes_per_elem, sharded=False, fused=None, n_buckets=None):
    """`config` of the JSON line -- identical keys (and values) for both arms, so the driver can match them."""
    c = wl.update_freq
    if fused is None:
        fused = world == 1 and args.fuse_final == 1 and not args.accum_fp32
    if n_buckets is None:
        n_buckets = plan_buckets_host(wl.numel, int(args.bucket_mib * (1 << 20)))
    return {"workload": wl.name, "n_params": wl.n, "n_tensors": len(wl.numel), "update_freq": c, "world": world,
            "bucket_mib": args.bucket_mib, "n_buckets": n_buckets, "tokens_per_update": int(toks_per_update),
            "generator": {"real": "G_real", "exact": "G_exact", "zero": "zeros",
                          "real_sparse": "G_real + row-sparse embedding"}[args.generator] + " (SURVEY 8(d.2))",
            "parallelism": f"dp{world}", "fuse_final": int(fused), "accum_fp32": int(args.accum_fp32),
            "path_bytes_per_elem": path_bytes_per_elem,
            "optimizer": "sharded (SURVEY f2)" if (sharded and world > 1) else "replicated (paper)",
            "ar_copy_engine": int(getattr(args, "ar_copy_engine", 0) or 0), "ar_pieces": int(getattr(args, "ar_pieces", 1) or 1),
            "l2": "inputs (c x 2n B + 16n B state) >> 126 MB L2; no flush"}


def path_bpe(c, world, fused, acc32):
    """Algorithmic HBM bytes per parameter of one update."""
    if fused:
        return (4 if c > 1 else 0) + 6 * max(c - 2, 0) + (30 if c > 1 else 28)
    if acc32:
        return 6 + 10 * (c - 2) + 8 + 28 if c > 1 else 32
    return 4 + 6 * (c - 1) + 28


def run_reference(args):
    """This tier's reference arm: the CPU oracle as it stands, on the box's host cores.  Each step is one whole
    oracle update (all c micro-batches of all W ranks, emulated) over a bounded contiguous slice of the workload's
    parameter vector, sized so the whole --steps/--warmup run takes about --ref-seconds; `ms_per_step` is the
    measured wall time of such a step, so ms_per_step x steps is what actually ran.  `value` = grad elements per
    second of those steps (the metric's unit); the full-vector update time is extrapolated beside it, labelled."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = set_generator(workload(args.config, args.gpus, args.update_freq), args.generator)
    W, c = wl.world, wl.update_freq
    # probe: one update on a small slice gives the oracle's rate; then size the slice for the budget
    probe_v, probe_s, _ = oracle_rate(wl, 0.0, slice_elems=min(wl.n, 1 << 18))
    per_step = max(0.05, args.ref_seconds / max(1, args.steps + args.warmup))
    slice_elems = int(min(wl.n, max(1 << 16, probe_v * per_step / (W * c))))
    for _ in range(args.warmup):
        oracle_rate(wl, 0.0, slice_elems=slice_elems)
    vals, secs = [], []
    for _ in range(args.steps):
        v, sec, sample = oracle_rate(wl, 0.0, slice_elems=slice_elems)
        vals.append(v)
        secs.append(sec)
    value = statistics.median(vals)
    fused = W == 1 and args.fuse_final == 1 and not args.accum_fp32
    toks = sum(synth_ntokens(wl, 1, r, k) for r in range(W) for k in range(1, c + 1))
    cfg = bench_config(args, wl, W, toks, path_bpe(c, W, fused, args.accum_fp32 and c > 1))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+binary16",
            "data": "synthetic", "config": cfg,
            "step_is": f"one whole oracle update over elements [0, {slice_elems}) of {wl.n} (all {W}x{c} "
                       f"micro-batches), not the full vector",
            "full_update_ms_extrapolated": 1000 * W * c * wl.n / value,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": omp_threads(), "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def synth_ntokens(wl, u, r, k):
    import synth
    return synth.ntokens(wl, u, r, k)


# ------------------------------------------------------------------------------------------ M2 backward load
class BackwardEmulator:
    """Timing-mode producer: per micro-batch of T target tokens, cuBLAS fp16 GEMMs of every
    weight matrix's real shape -- forward Y = X W^T, backward dX = dY W and dW = dY^T X (6 n T flops) -- on the
    library's own fp16 weights (smpu_weights_fp16, "forward-backward computations ... in FP16").
    Backward runs in gradient-ready order; `on_bucket(b)` fires once the last tensor of bucket b has its
    dW, which is when the paper adds it to the synchronisation buffer.  Gradient VALUES still come from
    the synthetic generator: the GEMMs emulate the load the all-reduce must hide behind, nothing more."""

    def __init__(self, wl, w16_ptr, bucket_begin, device, t_max=3500):
        import torch
        n = wl.n

        class _View:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f2", "data": (ptr, False),
                                                 "version": 3}
        w16 = torch.as_tensor(_View(w16_ptr, n), device=device)
        d = None
        for name, numel, _ in wl.tensors:
            if name.endswith("in_proj.weight"):
                d = int(round((numel // 3) ** 0.5))
                break
        self.mats = []          # (ready index, out, in, view) for every weight matrix
        off = 0
        for j, (name, numel, cls) in enumerate(wl.tensors):
            if name.endswith(".weight") and numel % d == 0 and numel // d > 1 and "ln" not in name.split(".")[-2]:
                rows = numel // d
                if name.endswith("fc2.weight"):
                    shape = (d, numel // d)
                else:
                    shape = (rows, d)
                self.mats.append((j, shape[0], shape[1], w16[off:off + numel].view(shape)))
            off += numel
        self.tensor_end = np.cumsum(wl.numel)
        self.bucket_of_end = {}
        # bucket b is complete once the tensor ending at bucket_begin[b+1] is done
        ends = {int(e): j for j, e in enumerate(self.tensor_end)}
        for b in range(len(bucket_begin) - 1):
            self.bucket_of_end[ends[int(bucket_begin[b + 1])]] = b
        dmax = max(max(o, i) for _, o, i, _ in self.mats)
        self.x = torch.randn(t_max, dmax, device=device, dtype=torch.float16) * 0.1
        self.dy = torch.randn(t_max, dmax, device=device, dtype=torch.float16) * 0.1
        self.out = torch.empty(t_max * dmax, device=device, dtype=torch.float16)
        self.dw = torch.empty(max(o * i for _, o, i, _ in self.mats), device=device, dtype=torch.float16)
        self.n_tensors = len(wl.tensors)
        self.flops_per_token = 6 * sum(o * i for _, o, i, _ in self.mats)
        self.offsets = np.concatenate([[0], np.cumsum(wl.numel)])
        # 1-D tensors (biases, LayerNorm) of the in-place producer: one indexed fp16 add per micro-batch
        mat_ids = {j for j, _, _, _ in self.mats}
        idx = [np.arange(self.offsets[j], self.offsets[j + 1]) for j in range(len(wl.tensors)) if j not in mat_ids]
        self.idx1d = torch.from_numpy(np.concatenate(idx).astype(np.int64)).to(device)
        self.one_d = [j for j in range(len(wl.tensors)) if j not in mat_ids]
        # issued right before the first bucket boundary, so that every bucket is complete when announced
        self.first_1d_ready = min(self.bucket_of_end) if self.bucket_of_end else 0
        self.vec1d = torch.randn(self.idx1d.numel(), device=device, dtype=torch.float16) * 0.01

    def micro(self, T, on_bucket=None, acc=None, first=False, on_tensor=None):
        """acc (the library's accumulator viewed as fp16[n]): accumulate in place instead of into scratch --
        dW GEMMs with beta = 0 (first micro-batch of the update) or 1, 1-D tensors by fp16 copy / add."""
        import torch
        x, dy = self.x[:T], self.dy[:T]
        for j, o, i, W in reversed(self.mats):                       # forward: reverse ready order
            torch.mm(x[:, :i], W.t(), out=self.out[:T * o].view(T, o))
        by_tensor = {j: (o, i, W) for j, o, i, W in self.mats}
        for j in range(self.n_tensors):                              # backward: ready order
            if j in by_tensor:
                o, i, W = by_tensor[j]
                torch.mm(dy[:, :o], W, out=self.out[:T * i].view(T, i))                    # dX
                if acc is not None:
                    dst = acc[self.offsets[j]:self.offsets[j + 1]].view(o, i)
                    torch.addmm(dst, dy[:, :o].t(), x[:, :i], beta=0.0 if first else 1.0, out=dst)
                else:
                    torch.mm(dy[:, :o].t(), x[:, :i], out=self.dw[:o * i].view(o, i))      # dW
            if acc is not None and j == self.first_1d_ready:
                # every 1-D tensor's gradient at once (they are tiny): copy or fp16 add at their indices
                acc.index_copy_(0, self.idx1d, self.vec1d) if first else acc.index_add_(0, self.idx1d, self.vec1d)
            if on_tensor is not None:                     # per-tensor ready hook
                if j == self.first_1d_ready:
                    for jj in self.one_d:                  # the 1-D tensors were all added just above
                        on_tensor(jj)
                if j not in self.one_d:
                    on_tensor(j)
            if on_bucket is not None and j in self.bucket_of_end:
                on_bucket(self.bucket_of_end[j])


def run_m2(args, P, wl, lay, grads, toks, step, stream, world, rank, local, cfg, theta0):
    """Whole training-step emulation: c micro-batches of backward load + the update step (library)."""
    import torch
    c = wl.update_freq

    def emulator_for(st):
        return BackwardEmulator(wl, st.weights_fp16_ptr(), st.bucket_begin, f"cuda:{local}")

    class _Acc:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f2", "data": (ptr, False), "version": 3}

    def one(st, emu):
        bb = st.bucket_begin
        if args.m2_fused:      # the backward accumulates in place; the library is told with None
            acc = torch.as_tensor(_Acc(st.accumulator_ptr(), lay.n), device=f"cuda:{local}")
            for k in range(c - 1):
                emu.micro(toks[k], acc=acc, first=(k == 0))
                st.accumulate(None, toks[k], stream)
            st.micro_begin(toks[c - 1])
            emu.micro(toks[c - 1], on_tensor=lambda j: st.tensor_ready(j, stream), acc=acc, first=(c == 1))
            st.step(stream, wait=False)
            return
        for k in range(c - 1):
            emu.micro(toks[k])
            st.accumulate(grads[k], toks[k], stream)
        st.micro_begin(toks[c - 1])
        emu.micro(toks[c - 1], on_bucket=lambda b: st.accumulate_bucket(b, grads[c - 1][bb[b]:bb[b + 1]], stream))
        st.step(stream, wait=False)

    def timed(st, emu, steps):
        for _ in range(args.warmup):
            one(st, emu)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            one(st, emu)
        b.record(stream)
        torch.cuda.synchronize()
        return _max_over_ranks(a.elapsed_time(b) / steps, world)

    emu = emulator_for(step)
    step.kernel_stats(reset=True)
    step.set_timing(True)
    ms = timed(step, emu, args.steps)
    step.set_timing(False)
    stats = step.kernel_stats(reset=True)
    # the same per-GPU work with no communication: a world = 1 ctx on the same GPU
    ms1 = None
    if world > 1:
        s1 = P.UpdateStep(wl.numel, theta0, cfg, world=1, rank=0, device=local)
        ms1 = timed(s1, emulator_for(s1), args.steps)
        s1.close()
    if rank != 0:
        return None
    tok_per_update = world * sum(toks)
    out = {"metric": METRIC + " (M2: with emulated backward)", "mode": "m2", "n_gpus": world,
           "producer": "in-place dW-GEMM accumulation (f3)" if args.m2_fused else "separate K1 accumulate",
           "target_tokens_per_s": tok_per_update / (ms * 1e-3),
           "ms_per_step": ms, "steps": args.steps, "warmup": args.warmup,
           "value": world * c * lay.n / (ms * 1e-3), "unit": UNIT,
           "config": {"workload": wl.name, "update_freq": c, "bucket_mib": args.bucket_mib,
                      "allreduce": {0: None, 1: "nccl", 2: "fused_lsa"}[step.allreduce_impl if world > 1 else 0],
                      "tokens_per_micro": toks, "backward_flops_per_update": emu.flops_per_token * sum(toks)},
           # CUDA-event brackets around the library's launches; with ~6,400 GEMM launches per update the host can
           # fall behind the GPU, and an enqueue gap then counts into the bracket: an upper bound
           "update_path_kernels_ms_per_step_upper_bound": (stats["k1_add"]["ms"] + stats["k1_first"]["ms"] + stats["k1s_sweep"]["ms"]
                                               + stats["k2_adam"]["ms"]) / (args.steps + args.warmup),
           "allreduce_ms_per_step": stats["allreduce"]["ms"] / args.steps}
    if ms1 is not None:
        out["exposed_comm"] = {"ms": ms - ms1, "frac_of_update": (ms - ms1) / ms, "t_world1_ms": ms1,
                               "method": "T(M2 step, W ranks) - T(same per-GPU M2 step through a world=1 ctx)"}
    return out


# ------------------------------------------------------------------------------------------ train (real producer)
def run_train(args, P, wl, lay, step, stream, world, rank, local, make_cfg, theta0):
    """SURVEY f3 with a real producer: each micro-batch is a forward + backward of the paper's Transformer-big
    (producer/transformer.py) on the library's fp16 weights, scaled by the library's loss scale; the first c - 1
    micro-batches go to smpu_accumulate after their backward, the last one bucket by bucket from the backward's
    per-tensor hooks -- or, with --no-overlap, after its backward.  Timed: whole training updates
    (c x fwd/bwd + the update step), CUDA events, max over ranks; exposed communication against the same producer
    through a world = 1 ctx."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "producer"))
    from transformer import GraphedProducer, Producer, TransformerBig, device_view
    c, n = wl.update_freq, lay.n
    side = torch.cuda.Stream(device=f"cuda:{local}")
    dropout = 0.1 if "enfr" in wl.name else 0.3

    def setup(st, seed):
        w16 = device_view(st.weights_fp16_ptr(), n, "<f2", f"cuda:{local}")
        scale = device_view(st.loss_scale_ptr(), 1, "<f4", f"cuda:{local}")
        model = TransformerBig(wl.tensors, w16, dropout=dropout)
        grad = torch.empty(n, dtype=torch.float16, device=f"cuda:{local}")
        prod = Producer(model, grad, scale, seed=seed)
        batches = [prod.batch(args.tokens, args.sent_len) for _ in range(c)]
        return prod, grad, batches

    def bucket_of(st):
        bb = st.bucket_begin
        tb = [int(np.searchsorted(bb, off, side="right") - 1) for off in np.concatenate([[0], np.cumsum(wl.numel)[:-1]])]
        per = np.bincount(tb, minlength=len(bb) - 1)
        return tb, per, bb

    def one(st, prod, grad, batches, overlap, gp=None):
        g16 = grad.view(torch.int16)
        if gp is not None:
            # graphed producer: the backward records each bucket's completion as an event inside its graph; the
            # library takes bucket b on a second stream as soon as that event fires
            for k in range(c - 1):
                src, ti, to, nt = batches[k]
                gp.micro(src, ti, to)
                st.accumulate(g16, nt, stream)
            src, ti, to, nt = batches[c - 1]
            events, _ = gp.micro(src, ti, to)
            if not overlap:
                st.accumulate(g16, nt, stream)
                st.step(stream, wait=False)
                return
            tb, per, bb = bucket_of(st)
            st.micro_begin(nt)
            for b in range(len(bb) - 1):
                side.wait_event(events[b])
                st.accumulate_bucket(b, g16[int(bb[b]):int(bb[b + 1])], side)
            st.step(side, wait=False)
            stream.wait_stream(side)          # the next replay rewrites the gradient buffer and reads w16
            return
        for k in range(c - 1):
            src, ti, to, nt = batches[k]
            prod.micro(src, ti, to)
            st.accumulate(g16, nt, stream)
        src, ti, to, nt = batches[c - 1]
        if not overlap:
            prod.micro(src, ti, to)
            st.accumulate(g16, nt, stream)
        else:
            tb, per, bb = bucket_of(st)
            left = per.copy()
            st.micro_begin(nt)

            def on_tensor(j):
                b = tb[j]
                left[b] -= 1
                if left[b] == 0:      # the bucket's last gradient is in: hand it over now
                    st.accumulate_bucket(b, g16[int(bb[b]):int(bb[b + 1])], stream)
            prod.micro(src, ti, to, on_tensor=on_tensor)
        st.step(stream, wait=False)

    def timed(st, w, overlap, seed):
        prod, grad, batches = setup(st, seed)
        gp = None
        if not args.eager_producer:
            tb, per, bb = bucket_of(st)
            gp = GraphedProducer(prod, tb, len(bb) - 1)
        for _ in range(max(1, args.warmup)):
            one(st, prod, grad, batches, overlap, gp)
        torch.cuda.synchronize()
        _barrier(w)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as clk:
            a.record(stream)
            for _ in range(args.steps):
                one(st, prod, grad, batches, overlap, gp)
            b.record(stream)
            torch.cuda.synchronize()
        _barrier(w)
        last = st.result(st.scalars()["attempts"])
        ms = a.elapsed_time(b) / args.steps
        return _max_over_ranks(ms, w), sum(x[3] for x in batches), last, clk.summary(), prod.flops_per_token()

    overlap = not args.no_overlap
    ms, tok_rank, last, clk, fpt = timed(step, world, overlap, seed=rank)
    ms_no = None
    if world > 1 and overlap:
        ms_no = timed(step, world, False, seed=rank)[0]
    step.close()
    ms1 = None
    if world > 1:
        s1 = P.UpdateStep(wl.numel, theta0, make_cfg(False, fuse_final=0), world=1, rank=0, device=local)
        ms1 = timed(s1, 1, False, seed=rank)[0]
        ms1 = _max_over_ranks(ms1, world)
        s1.close()
    tok = _sum_over_ranks(tok_rank, world)
    if rank != 0:
        return None
    out = {"metric": METRIC + " (train: real Transformer-big forward/backward producer)", "mode": "train",
           "value": world * c * n / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "target_tokens_per_s": tok / (ms * 1e-3), "tokens_per_update": tok, "update_freq": c,
           "model_flops_per_token": fpt, "model_tflops_per_s_per_gpu": fpt * tok / world / (ms * 1e-3) / 1e12,
           "last_result": {k: last[k] for k in ("applied", "overflow", "scale_log2_used", "lr", "num_updates")},
           "overlap": "per-bucket handover from backward hooks (P:211-212)" if overlap else "after backward",
           "producer_mode": "eager" if args.eager_producer else "CUDA graph per batch shape (bucket events in-graph)",
           "config": {"workload": wl.name, "update_freq": c, "world": world, "bucket_mib": args.bucket_mib,
                      "tokens_per_micro_budget": args.tokens, "sent_len": args.sent_len, "dropout": dropout,
                      "label_smoothing": 0.1, "data": "synthetic uniform token ids (no dataset)",
                      "producer": "producer/transformer.py (torch fp16 autograd on the library's w16)"},
           "clocks": clk, "dtype": "f16+f32", "data": "synthetic"}
    if ms1 is not None:
        out["exposed_comm"] = {"ms": ms - ms1, "frac_of_update": (ms - ms1) / ms, "t_world1_ms": ms1,
                               "method": "T(training update, W ranks) - T(same producer + world=1 ctx, same GPU)"}
    if ms_no is not None:
        out["no_overlap_ms_per_step"] = ms_no
        out["overlap_gain"] = (ms_no - ms) / ms_no
    return out


# ------------------------------------------------------------------------------------------ our arm
def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def own_launches(stats, ar_impl, nccl_impl):
    """Kernels of libsmpu.so in `stats` (every kind, except the all-reduces when NCCL runs them)."""
    lib_kinds = ("allreduce", "decision_ar") if ar_impl == nccl_impl else ()
    return int(sum(v["launches"] for k, v in stats.items() if k not in lib_kinds))


_TRACE_N = [0]


def measure(args, step, grads, toks, stream, world, local, resident=True):
    """Time one ctx: a call-by-call region (kernel events -> per-kernel table, roofline) and the captured CUDA graph of
    the same update (the headline unless --no-graph), each after warm-up and a ~0.6 s soak under the clock sampler,
    bracketed by barrier + synchronize, CUDA events on the launch stream, max over ranks."""
    import torch
    c = len(grads)

    def one_update():
        for k in range(c):
            step.accumulate(grads[k], toks[k], stream)
        step.step(stream, wait=False)

    t_w = time.perf_counter()
    for _ in range(args.warmup):
        one_update()
    torch.cuda.synchronize()
    per_update = _max_over_ranks((time.perf_counter() - t_w) / max(1, args.warmup), world)
    soak = max(2, min(2000, int(0.6 / max(per_update, 1e-5))))     # same count on every rank (collectives)
    _barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        for _ in range(soak):
            one_update()
        step.kernel_stats(reset=True)
        step.set_timing(True)
        torch.cuda.synchronize()
        _barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            one_update()
        ev1.record(stream)
        torch.cuda.synchronize()
        _barrier(world)
    step.set_timing(False)
    out = {"ms_calls": ev0.elapsed_time(ev1) / args.steps, "clk": clk}
    out["ms"] = out["ms_calls"]
    if args.trace:
        # one file per timed ctx of the run (headline, sharded variant, world = 1 baseline ...), per rank
        _TRACE_N[0] += 1
        with open(f"{args.trace}.{_TRACE_N[0]}" + ("" if world == 1 else f".rank{step.rank}"), "w") as f:
            for kname, sname, a, b in step.kernel_trace():
                f.write(json.dumps({"rank": step.rank, "kernel": kname, "stream": sname, "start_ms": round(a, 4),
                                    "end_ms": round(b, 4)}) + "\n")
    out["stats"] = step.kernel_stats(reset=True)
    last = step.result(step.scalars()["attempts"])
    assert last["applied"] == 1 and last["overflow"] == 0, last
    out["graph"] = None
    if args.no_graph:
        return out
    import paper_1806_00187_b200 as P
    try:
        step.graph_capture(grads)
    except P.SmpuError as ex:          # e.g. W > 1 fell back to NCCL (not graph-capturable here)
        print(f"[bench] graph capture unavailable ({ex}); timing the call-by-call path", file=sys.stderr)
        return out
    for _ in range(args.warmup):
        step.graph_launch(toks, stream)
    torch.cuda.synchronize()
    _barrier(world)
    with Clocks(local) as clk_g:
        for _ in range(soak):
            step.graph_launch(toks, stream)
        step.kernel_stats(reset=True)
        torch.cuda.synchronize()
        _barrier(world)
        # an event after every replay on the launch stream: the per-update distribution (SURVEY d.4 p10/p50/p90)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev0.record(stream)
        for i in range(args.steps):
            step.graph_launch(toks, stream)
            marks[i].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        _barrier(world)
    out["ms"] = ev0.elapsed_time(ev1) / args.steps
    per = np.diff([0.0] + [ev0.elapsed_time(m) for m in marks])
    out["per_update_ms"] = {"p10": float(np.percentile(per, 10)), "p50": float(np.percentile(per, 50)),
                            "p90": float(np.percentile(per, 90)), "max": float(per.max()), "n": int(per.size)}
    out["gstats"] = step.kernel_stats(reset=True)
    out["clk"] = clk_g
    last = step.result(step.scalars()["attempts"])
    assert last["applied"] == 1 and last["overflow"] == 0, last
    out["graph"] = {"ms_per_step_graph": out["ms"], "ms_per_step_calls": out["ms_calls"]}
    if resident:
        # variant: the producer keeps all c micro-batch gradients resident (6.7 GB of 180 GB) and the update
        # accumulates them in one pass (smpu_accumulate_many; bitwise the same sums) -- reported beside the
        # headline, which keeps the paper's in-place accumulation after every micro-batch
        step.graph_capture(grads, resident=True)
        for _ in range(args.warmup):
            step.graph_launch(toks, stream)
        torch.cuda.synchronize()
        _barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            step.graph_launch(toks, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        _barrier(world)
        out["ms_resident"] = _max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
        last = step.result(step.scalars()["attempts"])
        assert last["applied"] == 1 and last["overflow"] == 0, last
    return out


def bus_gbs(stats, steps, n, world, sharded):
    """In-situ bus bandwidth of the bucket all-reduce (nccl-tests convention): all-reduce 2(W-1)/W x 2n bytes per
    update; the sharded layout's timed kernel is the reduce-scatter alone, (W-1)/W x 2n (its w16 all-gather is peer
    stores inside the Adam kernel)."""
    ar_ms = stats["allreduce"]["ms"] / steps
    if ar_ms <= 0:
        return None
    phases = 1 if sharded else 2
    bus = phases * n * 2 * (world - 1) / world / (ar_ms * 1e-3) / 1e9
    return {"ms_per_step": ar_ms, "bus_gbs": bus, "frac_of_900": bus / NVLINK_NOMINAL_GBS,
            "frac_of_measured_nvlink": bus / NVLINK_MEASURED_GBS, "measured_nvlink_gbs": NVLINK_MEASURED_GBS,
            "in_situ": "concurrent with K1 / Adam"}


def bind_to_gpu_numa(local):
    """Run this rank on the CPUs NVML lists as local to its GPU, so that its pinned host buffers (the e2e inputs,
    first-touch allocated by cudaHostAlloc) sit on the GPU's NUMA node.  Returns the CPU count, or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        cpus &= set(range(os.cpu_count() or 1))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        return None
    return None


def main_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    numa_cpus = bind_to_gpu_numa(local) if world > 1 else None
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1806_00187_b200 as P
    import synth

    wl = set_generator(workload(args.config, world, args.update_freq), args.generator)
    lay = synth.Layout(wl)
    c, n = wl.update_freq, lay.n

    def new_id():
        if world == 1:
            return None
        obj = [P.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    # inputs resident in HBM: theta_0 and c micro-gradient buffers of this rank (update u = 1, e = 7)
    theta0 = torch.empty(n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    grads = []
    for k in range(1, c + 1):
        g = torch.empty(n, dtype=torch.int16, device="cuda")
        synth.micro_grad_gpu(g, wl, lay, 1, rank, k, 7)
        grads.append(g)
    toks = [synth.ntokens(wl, 1, rank, k) for k in range(1, c + 1)]
    toks_all = _sum_over_ranks(sum(toks), world)
    # the headline layout: the paper's replicated update; --optimizer sharded makes f2 the headline
    head_sharded = world > 1 and (args.optimizer == "sharded" or args.sharded)
    ar = {"auto": 0, "nccl": 1, "fused": 2}[args.allreduce]

    def make_cfg(sharded, fuse_final=args.fuse_final):
        cfg = P.config_default(update_freq=c, bucket_bytes=int(args.bucket_mib * (1 << 20)), allreduce=ar,
                               sharded=int(sharded), fuse_final=fuse_final, accum_fp32=int(args.accum_fp32),
                               ar_ctas=args.ar_ctas, ar_unroll=args.ar_unroll, ar_threads=args.ar_threads)
        if args.ar_pieces is not None:
            cfg.ar_pieces = args.ar_pieces
        if not sharded:
            cfg.ar_copy_engine = args.ar_copy_engine
        # growth interval beyond the run: the scale stays at 2^7, so the pre-generated inputs stay valid
        cfg.growth_interval = 1 << 40
        return cfg

    fused = world == 1 and args.fuse_final == 1 and not args.accum_fp32
    acc32 = args.accum_fp32 and c > 1
    torch.cuda.synchronize()
    cfg = make_cfg(head_sharded)
    step = P.UpdateStep(wl.numel, theta0, cfg, world=world, rank=rank, nccl_id=new_id(), device=local)
    ar_impl = step.allreduce_impl
    stream = torch.cuda.current_stream()
    if args.mode in ("m2", "train"):
        if args.mode == "m2":
            out = run_m2(args, P, wl, lay, grads, toks, step, stream, world, rank, local, cfg, theta0)
            step.close()
        else:
            del grads
            out = run_train(args, P, wl, lay, step, stream, world, rank, local, make_cfg, theta0)
        if out is not None:
            emit(out)
        if world > 1:
            dist.destroy_process_group()
        return

    M = measure(args, step, grads, toks, stream, world, local)
    ms, ms_calls, stats = M["ms"], M["ms_calls"], M["stats"]
    nb = step.n_buckets
    shard = sum(h - l for l, h in step.shard_ranges())

    # ---- end-to-end through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        pool = min(c, 4)
        host = [grads[k].cpu().pin_memory() for k in range(pool)]
        torch.cuda.synchronize()
        _barrier(world)
        for k in range(c):
            step.accumulate(host[k % pool], toks[k], stream)
        step.step(stream, wait=True)
        _barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            for k in range(c):
                step.accumulate(host[k % pool], toks[k], stream)
            step.step(stream, wait=True)          # device -> host read of the step's result
        e2e_s = _max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, world)
        e2e = {"value": world * c * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": c * n * 2,
               "d2h_bytes_per_step": ctypes_sizeof_result(), "ms_per_step": 1000 * e2e_s,
               "source": "pinned host fp16 micro-gradients, staged H2D inside smpu_accumulate",
               "rank_cpus_numa_local": numa_cpus}
        del host
    # ---- the bucket all-reduce standalone (SURVEY d.4: "measure it standalone ... and in situ"): the headline ctx's
    # smpu_allreduce_accumulator back to back, CUDA events, max over ranks (its values are overwritten by the next
    # update's first K1; nothing else reads them)
    ar_alone = None
    if world > 1 and ar_impl == P.smpu.AR_FUSED and not head_sharded:
        for _ in range(3):
            step.allreduce_accumulator(stream)
        torch.cuda.synchronize()
        _barrier(world)
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        for _ in range(10):
            step.allreduce_accumulator(stream)
        b_ev.record(stream)
        torch.cuda.synchronize()
        _barrier(world)
        t_ar = _max_over_ranks(a_ev.elapsed_time(b_ev) / 10, world)
        bus = 2 * n * 2 * (world - 1) / world / (t_ar * 1e-3) / 1e9
        ar_alone = {"ms": t_ar, "bus_gbs": bus, "frac_of_900": bus / NVLINK_NOMINAL_GBS,
                    "frac_of_measured_nvlink": bus / NVLINK_MEASURED_GBS,
                    "launches": step.n_buckets * args.ar_pieces,
                    "what": "smpu_allreduce_accumulator back to back (every bucket, the headline's ar_pieces)"}
    step.close()
    del step

    # ---- W = 1: the opt-in fused last micro-batch (smpu_config.fuse_final = 1) beside the contract-default headline
    fused_variant = None
    if world == 1 and not fused and not args.accum_fp32:
        fstep = P.UpdateStep(wl.numel, theta0, make_cfg(False, fuse_final=1), world=1, rank=0, device=local)
        F_ = measure(args, fstep, grads, toks, stream, 1, local, resident=True)
        fb = (4 if c > 1 else 0) + 6 * max(c - 2, 0) + (30 if c > 1 else 28)
        k12 = F_["stats"]["k12_fused"]
        fused_variant = {"ms_per_step": F_["ms"], "value": c * n / (F_["ms"] * 1e-3), "bytes_per_elem": fb,
                         "path_hbm_gbs": fb * n / (F_["ms"] * 1e-3) / 1e9,
                         "k12_achieved_gbs": (30 if c > 1 else 28) * n * k12["launches"] / max(1, k12["launches"]) /
                                             (k12["ms"] / max(1, k12["launches"]) * 1e-3) / 1e9 if k12["ms"] > 0 else None,
                         "resident_ms_per_step": F_.get("ms_resident"),
                         "api": "smpu_config.fuse_final = 1 (opt-in; w16 rewritten by the last accumulate call)"}
        fstep.close()
        del fstep

    # ---- W > 1: the sharded layout beside the replicated headline, same inputs
    variant = None
    if world > 1 and not head_sharded and args.optimizer == "auto" and ar_impl == P.smpu.AR_FUSED:
        sstep = P.UpdateStep(wl.numel, theta0, make_cfg(True), world=world, rank=rank, nccl_id=new_id(), device=local)
        V = measure(args, sstep, grads, toks, stream, world, local, resident=False)
        variant = {"ms_per_step": _max_over_ranks(V["ms"], world), "ms_per_step_calls": _max_over_ranks(V["ms_calls"], world),
                   "allreduce": bus_gbs({k: {"ms": _max_over_ranks(v["ms"], world)} for k, v in V["stats"].items()},
                                        args.steps, n, world, True),
                   "shard_elems": sum(h - l for l, h in sstep.shard_ranges())}
        variant["value"] = world * c * n / (variant["ms_per_step"] * 1e-3)
        variant["update_steps_per_s"] = 1000.0 / variant["ms_per_step"]
        sstep.close()
        del sstep

    # ---- exposed communication: the same per-GPU work through a world = 1 ctx on the same GPU (fuse_final = 0:
    # the W > 1 kernels -- accumulate, decide, Adam over all n -- minus the exchange)
    t1 = k2_full_ms = None
    if world > 1:
        step1 = P.UpdateStep(wl.numel, theta0, make_cfg(False, fuse_final=0), world=1, rank=0, device=local)
        B = measure(args, step1, grads, toks, stream, 1, local, resident=False)
        t1 = _max_over_ranks(B["ms"], world)
        k2_full_ms = _max_over_ranks(B["stats"]["k2_adam"]["ms"] / args.steps, world)
        step1.close()
        del step1

    ms = _max_over_ranks(ms, world)
    ms_calls = _max_over_ranks(ms_calls, world)
    kstat = {k: {"launches": v["launches"], "ms": _max_over_ranks(v["ms"], world)} for k, v in stats.items()}
    ms_res = M.get("ms_resident")
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    hbm_peak = peaks["hbm_gbs"] if peaks else 6650.0
    peak_src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if peaks else "of fallback (B200_PROFILING.md)"
    # algorithmic bytes per launch: K1 first 4 B/elem, K1 add 6, K1s 2, K2 28, K12 (the
    # fused last micro-batch + Adam, W = 1) 30 (28 at c = 1: no accumulator read)
    # (K1s only sweeps when the early decision was undecided; with G_real it returns at once)
    # with the fp32 accumulator (Z1 knob): first 6 B/elem, add 10, the last micro-batch 8 (rn16 into acc16)
    if fused:
        step_bytes = {"k1_first": 4 * n if c > 1 else 0, "k1_add": 6 * max(c - 2, 0) * n, "k2_adam": 0,
                      "k12_fused": (30 if c > 1 else 28) * n}
    elif acc32:
        step_bytes = {"k1_first": 6 * n, "k1_add": (10 * (c - 2) + 8) * n, "k2_adam": 28 * shard, "k12_fused": 0}
    else:
        step_bytes = {"k1_first": 4 * n, "k1_add": 6 * (c - 1) * n, "k2_adam": 28 * shard, "k12_fused": 0}
    kernels = {}
    for k, per_step in step_bytes.items():
        st = kstat[k]
        if st["launches"] == 0 or st["ms"] <= 0 or per_step == 0:
            continue
        bytes_total = per_step * args.steps
        kernels[k] = {"launches": st["launches"], "avg_us": 1000 * st["ms"] / st["launches"],
                      "share_of_step": st["ms"] / (ms_calls * args.steps),
                      "algorithmic_bytes_per_launch": bytes_total / st["launches"],
                      "achieved_gbs": bytes_total / (st["ms"] * 1e-3) / 1e9}
    dom = max(kernels, key=lambda k: kernels[k]["share_of_step"])
    traffic = load_traffic(dom, wl.name)
    # second denominator for context: ncu's DRAM peak (dram__bytes.sum.peak_sustained 2048 B/cycle x 3.996 GHz)
    ncu_dram_peak = 2048 * 3.996
    roof = {"kernel": dom, "bound": "hbm", "achieved": kernels[dom]["achieved_gbs"], "peak": hbm_peak,
            "unit": "GB/s", "frac": kernels[dom]["achieved_gbs"] / hbm_peak, "peak_source": peak_src,
            "traffic": traffic, "frac_of_ncu_dram_peak": kernels[dom]["achieved_gbs"] / ncu_dram_peak}
    path_bytes = sum(step_bytes.values())
    out = {"metric": METRIC, "value": world * c * n / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f16+f32", "data": "synthetic",
           "config": bench_config(args, wl, world, toks_all, path_bytes / n, sharded=head_sharded, fused=fused,
                                  n_buckets=nb),
           "update_steps_per_s": 1000.0 / ms,
           "path_hbm_gbs": path_bytes / (ms * 1e-3) / 1e9,
           "path_hbm_frac": path_bytes / (ms * 1e-3) / 1e9 / hbm_peak,
           "roofline": roof, "kernels": kernels,
           # our kernels in the timed region (the graph replays' when the graph is timed)
           "gpu_launches": own_launches(M["gstats"] if M["graph"] else stats, ar_impl, P.smpu.AR_NCCL),
           "clocks": M["clk"].summary(),
           "timed_path": "calls (c x smpu_accumulate + smpu_step)" if not M["graph"] else
                         "cuda_graph (smpu_graph_launch of the captured update; kernels/roofline from the call path)"}
    if M["graph"]:
        g = dict(M["graph"])
        if "per_update_ms" in M:
            g["per_update_ms_rank0"] = M["per_update_ms"]
        g["launches_per_step"] = own_launches(M["gstats"], ar_impl, P.smpu.AR_NCCL) / args.steps
        if ms_res:
            # one pass over the c gradients (+ the accumulator written, then Adam's 28) or, fused, straight into Adam
            res_bpe = (10 * c + 22) if acc32 else (2 * c + 26 if fused else 2 * c + 2 + 28)
            g["resident_microbatches"] = {
                "ms_per_step": ms_res, "value": world * c * n / (ms_res * 1e-3), "unit": UNIT,
                "path_hbm_gbs": n * res_bpe / (ms_res * 1e-3) / 1e9, "bytes_per_elem": res_bpe,
                "api": "smpu_graph_capture(..., SMPU_GRAPH_RESIDENT) -> one smpu_accumulate_many over c buffers"}
        out["graph"] = g
    if t1 is not None:
        out["exposed_comm"] = {"ms": ms - t1, "frac_of_update": (ms - t1) / ms, "t_world1_ms": t1,
                               "layout": "sharded (SURVEY f2)" if head_sharded else "replicated (paper)",
                               "method": "T(update, W ranks) - T(same per-GPU work through a world=1 ctx, same "
                                         "GPU, same run, fuse_final=0); library-only step (no backward to hide "
                                         "behind)"}
        if head_sharded:
            base = t1 - k2_full_ms * (1 - 1 / world)
            out["exposed_comm"].update(ms=ms - base, frac_of_update=(ms - base) / ms, t_world1_ms=base,
                                       method="estimate: world=1 time with its Adam share (CUDA events) scaled to "
                                              "the shard, 1/W of it")
    if world > 1:
        a = bus_gbs(kstat, args.steps, n, world, head_sharded)
        if a:
            a["impl"] = {1: "nccl", 2: "fused_lsa"}.get(ar_impl, str(ar_impl)) + ("_reduce_scatter" if head_sharded else "")
            if ar_alone:
                a["standalone"] = ar_alone
            out["allreduce"] = a
    if fused_variant:
        out["fused_final_variant"] = fused_variant
    if variant:
        base = t1 - k2_full_ms * (1 - 1 / world)
        variant["exposed_comm_estimate"] = {
            "ms": variant["ms_per_step"] - base, "frac_of_update": (variant["ms_per_step"] - base) / variant["ms_per_step"],
            "t_baseline_ms": base,
            "method": "T(sharded update, W ranks) - [T(world=1 ctx) - (1 - 1/W) x its Adam time]: the same per-GPU "
                      "work (K1 passes over n, Adam over n/W) without the exchange, estimated"}
        variant["layout"] = "sharded (SURVEY f2): reduce-scatter, Adam on 1/W, w16 all-gathered by peer stores; bitwise the replicated update (tests/test_gpu_virtual.py, test_gpu_multi.py)"
        out["sharded_variant"] = variant
    if e2e:
        out["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        import oracle as O
        cores = omp_threads()
        v, _, sample = oracle_rate(wl, args.cpu_seconds)
        # and on one thread (SURVEY 8(d.4) asks for both), on a shorter sample
        O.set_threads(1)
        v1, _, sample1 = oracle_rate(wl, max(2.0, args.cpu_seconds / 4))
        O.set_threads(cores)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                               "value_1_thread": v1, "sample_1_thread": sample1, "cpu_model": cpu_model()}
    emit(out)
    if world > 1:
        dist.destroy_process_group()


def ctypes_sizeof_result():
    import ctypes
    from paper_1806_00187_b200 import smpu
    return ctypes.sizeof(smpu.StepResult)


_JSON_OUT = None


def keep_stdout_for_json():
    """From here on, anything written to file descriptor 1 -- NCCL's C-level `NCCL version ...` banner included --
    goes to stderr; the one JSON line goes to the original stdout (emit), so the driver reads exactly one line."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(obj):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([int(x)], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    return int(t.item())


def spawn_ranks(args):
    """--gpus N > 1 without torchrun: launch N ranks of this same command, one process per GPU, on 127.0.0.1 (the
    environment torchrun would give them); rank 0 prints the line.  Exit status: the worst rank's."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rcs = [p.wait() for p in procs]
    bad = [rc for rc in rcs if rc != 0]
    sys.exit(bad[0] if bad else 0)


def load_traffic(kernel, workload_name):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload_name, {}).get(kernel)
    except Exception:
        return None


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)        # the ranks inherit the real stdout; rank 0 prints the line
        return
    keep_stdout_for_json()
    if args.impl == "reference":
        run_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
