#!/usr/bin/env python
"""Standalone bucket all-reduce bandwidth (SURVEY 8(d.4) "measure it standalone"): the library's fused
deterministic all-reduce and its NCCL path through smpu_allreduce_accumulator, and torch.distributed's NCCL
all_reduce of the same bytes as the library baseline; Transformer-big En-De buckets (3 x ~150 MiB, 420 MB).
torchrun --nproc-per-node N tools/ar_bench.py  -> rank 0 prints one JSON line per variant."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1806_00187_b200 as P  # noqa: E402
import synth  # noqa: E402
from synth import models  # noqa: E402


def timed(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = models.big_ende(world)
    n = wl.n
    theta0 = torch.zeros(n, dtype=torch.float32, device="cuda")
    out = []
    for name, ar in (("fused_lsa", P.smpu.AR_FUSED), ("nccl (library)", P.smpu.AR_NCCL)):
        obj = [P.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cfg = P.config_default(update_freq=1, allreduce=ar)
        st = P.UpdateStep(wl.numel, theta0, cfg, world=world, rank=rank, nccl_id=obj[0], device=local)
        ms = timed(lambda: st.allreduce_accumulator())
        out.append((name, ms, st.n_buckets))
        st.close()
    x = torch.zeros(n, dtype=torch.float16, device="cuda")
    ms = timed(lambda: dist.all_reduce(x))
    out.append(("torch.distributed nccl, one 420 MB tensor", ms, 1))
    if rank == 0:
        for name, ms, nb in out:
            bus = 2 * n * 2 * (world - 1) / world / (ms * 1e-3) / 1e9
            print(json.dumps({"world": world, "impl": name, "buckets": nb, "bytes": 2 * n, "ms": ms,
                              "bus_gbs": bus, "frac_of_900": bus / 900, "frac_of_measured_nvlink_675": bus / 675}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
