"""N > 1 host logic on CPU: world-size-2 `gloo` process groups (no GPU).

Covers what the multi-GPU path does outside the kernels: every rank derives the same bucket plan from the
host-only C ABI call; the NCCL unique id and scalars travel through torch.distributed; the fp16 cross-rank sum
of exactly-summable accumulators equals the oracle's ascending-rank reduce bitwise whatever the collective's
order (reading R3); the int64 token count is summed exactly; replicas that apply the same reduced
gradient hold bitwise identical state; bench.py's max-over-ranks timing reduction.
"""
import hashlib
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        import oracle as O
        import paper_1806_00187_b200 as P
        import synth
        from synth import models
        import bench

        # 1. identical bucket plans from the host-only ABI call
        wl = models.big_ende(world=world)
        plan = P.plan_buckets(wl.numel, 150 << 20).tolist()
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        out["plans_equal"] = all(p == plans[0] for p in plans)

        # 2. a 128-byte id from rank 0 reaches every rank unchanged (the NCCL unique-id path of bench.py)
        blob = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        out["id_ok"] = blob[0] == bytes(range(128))

        # 3. fp16 all-reduce of exactly-summable accumulators == oracle ascending-rank reduce, bitwise
        c = 4
        small = models.Workload("d", [("w", 50_000, 0), ("b", 999, 1), ("e", 7_000, 2)], world, c, family="exact",
                                injections=[dict(u=2, kind="RED_OVF", i=123)])
        lay = synth.Layout(small)
        orc = O.Oracle(synth.theta0_cpu(small, lay))
        hashes = []
        for u in (1, 2, 3):
            e = orc.e
            mine = O.accumulate([synth.micro_grad_cpu(small, lay, u, rank, k, e) for k in range(1, c + 1)])
            t = torch.from_numpy(mine.view(np.float16).copy())
            dist.all_reduce(t)
            R_coll = t.numpy().view(np.uint16)
            allA = [O.accumulate([synth.micro_grad_cpu(small, lay, u, r, k, e) for k in range(1, c + 1)])
                    for r in range(world)]
            R_orc = O.reduce(allA)
            fin = (R_orc & 0x7C00) != 0x7C00
            out[f"R_equal_{u}"] = bool(np.array_equal(R_coll[fin], R_orc[fin]) and
                                       np.array_equal(R_coll[~fin] & 0x7C00, R_orc[~fin] & 0x7C00))
            # 4. exact int64 token sum
            mytok = sum(synth.ntokens(small, u, rank, k) for k in range(1, c + 1))
            tt = torch.tensor([mytok], dtype=torch.int64)
            dist.all_reduce(tt)
            N = sum(synth.ntokens(small, u, r, k) for r in range(world) for k in range(1, c + 1))
            out[f"N_equal_{u}"] = int(tt.item()) == N
            # 5. every replica applies the same R -> identical state (the oracle's scaler + Adam on R_coll)
            res = orc.update([[R_coll]], [[N]])
            hashes.append(hashlib.sha256(orc.theta.tobytes() + orc.w16.tobytes()).hexdigest())
            out[f"overflow_{u}"] = res["overflow"]
        allh = [None] * world
        dist.all_gather_object(allh, hashes)
        out["replicas_equal"] = all(h == allh[0] for h in allh)

        # 6. bench.py's max-over-ranks reduction (gloo path)
        out["max"] = bench._max_over_ranks(float(rank + 1) * 1.5, world)
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        out["error"] = traceback.format_exc() + repr(ex)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_host_path(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 300
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, out in res.items():
        assert "error" not in out, out.get("error")
        assert out["plans_equal"] and out["id_ok"] and out["replicas_equal"]
        for u in (1, 2, 3):
            assert out[f"R_equal_{u}"], (r, u)
            assert out[f"N_equal_{u}"], (r, u)
        assert out["overflow_2"] == 1 and out["overflow_1"] == 0 and out["overflow_3"] == 0   # RED_OVF at u=2
        assert out["max"] == 1.5 * world
