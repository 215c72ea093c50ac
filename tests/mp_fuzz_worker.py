"""Randomised parity on REAL peers (one process per GPU, NCCL symmetric windows over NVLink): the W > 1 fuzz of
tests/test_gpu_virtual_fuzz.py through LsaPeers -- peer pointers, LSA barriers, the copy engines writing into the
other ranks' windows -- instead of local windows.  Every rank draws the same cases from one seeded generator; each
case is a fresh ctx (its own communicator): random tensor lists, update_freq 1..3, bucket thresholds 2 B..1 MiB,
SM / copy-engine / CE-but-last all-reduce, ar_pieces 1..3, replicated or sharded, injections on any rank; 3 updates,
decisions and R bitwise against the oracle (computed on every rank for all ranks), replicas' w16 identical.

usage (torchrun): tests/mp_fuzz_worker.py CASES SEED
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_1806_00187_b200 as P  # noqa: E402
import synth  # noqa: E402
from synth import models  # noqa: E402
from tests.gpu_util import decisions, h2t, lib_cfg, oracle_decisions  # noqa: E402


def draw_case(rng, W):
    nt = int(rng.integers(1, 5))
    tensors = [(f"t{j}", int(rng.integers(1, 30_000)), int(rng.integers(0, 3))) for j in range(nt)]
    n = sum(t[1] for t in tensors)
    c = int(rng.integers(1, 4))
    inj = []
    for u in (1, 2, 3):
        if rng.integers(0, 3) == 0:
            kinds = ["INF", "NINF", "NAN", "RED_OVF", "BIG"] + (["ACC_OVF"] if c >= 2 else [])
            kind = kinds[int(rng.integers(0, len(kinds)))]
            d = dict(u=u, kind=kind, i=int(rng.integers(0, n)))
            if kind in ("INF", "NINF", "NAN"):
                d.update(r=int(rng.integers(0, W)), k=int(rng.integers(1, c + 1)))
            elif kind == "ACC_OVF":
                d.update(r=int(rng.integers(0, W)))
            inj.append(d)
    sharded = bool(rng.integers(0, 4) == 0)
    ce = 0 if sharded else int(rng.integers(0, 3))
    pieces = 1 if sharded else int(rng.integers(1, 4))
    bucket_bytes = [2, 1000, 16_384, 100_000, 1 << 20][int(rng.integers(0, 5))]
    return tensors, c, inj, sharded, ce, pieces, bucket_bytes


def main():
    cases, seed = int(sys.argv[1]), int(sys.argv[2])
    rank, W = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rng = np.random.default_rng(seed)
    failures = []
    for case_id in range(cases):
        tensors, c, inj, sharded, ce, pieces, bucket_bytes = draw_case(rng, W)
        desc = (case_id, tensors, c, inj, sharded, ce, pieces, bucket_bytes)
        wl = models.Workload("mpfuzz", tensors, W, c, injections=inj)
        lay = synth.Layout(wl)
        theta0 = synth.theta0_cpu(wl, lay)
        obj = [P.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        step = P.UpdateStep(wl.numel, theta0 if rank == 0 else np.zeros_like(theta0),
                            lib_cfg(wl, bucket_bytes=bucket_bytes, allreduce=P.smpu.AR_FUSED, sharded=int(sharded),
                                    ar_copy_engine=ce, ar_pieces=pieces),
                            world=W, rank=rank, nccl_id=obj[0], device=local)
        ranges = step.shard_ranges() if sharded else [(0, lay.n)]
        orc = O.Oracle(theta0)
        e = 7
        for u in range(1, 4):
            grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, e) for k in range(1, c + 1)] for r in range(W)]
            toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(W)]
            for k in range(c):
                step.accumulate(h2t(grads[rank][k]), toks[rank][k])
            res = step.step()
            ores = orc.update(grads, toks)
            if decisions(res) != oracle_decisions(ores):      # keep going: every rank must run the same calls
                failures.append(f"{desc} u{u}: decisions {decisions(res)} vs {oracle_decisions(ores)}")
            acc = step.get_state(P.smpu.STATE_ACCUM)
            R = ores["R"]
            for lo, hi in ranges:
                g, r_ = acc[lo:hi], R[lo:hi]
                nan = np.isnan(r_.view(np.float16))
                if not (np.array_equal(np.isnan(g.view(np.float16)), nan) and np.array_equal(g[~nan], r_[~nan])):
                    failures.append(f"{desc} u{u}: R differs on [{lo}, {hi})")
                    break
            w16 = step.get_state(P.smpu.STATE_W16)
            allw = [None] * W
            dist.all_gather_object(allw, w16.tobytes())
            if len(set(allw)) != 1:
                failures.append(f"{desc} u{u}: replicas' w16 differ")
            e = res["scale_log2_next"]
        step.close()
    allf = [None] * W
    dist.all_gather_object(allf, failures)
    dist.destroy_process_group()
    flat = [f for x in allf for f in x]
    if flat:
        print("FAIL", *flat[:20], sep="\n")
        sys.exit(1)
    if rank == 0:
        print(f"mp fuzz ok: {cases} random cases at W = {W} (seed {seed})")


if __name__ == "__main__":
    main()
