"""Multi-GPU parity worker (launched by tests/test_gpu_multi.py under torch.distributed.run, one rank per GPU).

Each rank feeds its own micro-gradients (G_exact: exactly summable, so NCCL's reduction order cannot change
a bit, reading R3) through libsmpu.so with world = W; per-bucket NCCL all-reduces run inside the library.
Rank 0 emulates all W ranks in the oracle (ascending-rank fp16 reduce) and compares decisions and the
reduced gradient bitwise and theta/m/v/w16 within tolerance; every rank checks that all replicas hold
bitwise identical state after every update (P:55-57 synchronous data parallelism).
"""
import hashlib
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
from tests.gpu_util import (Magnitudes, check_state, decisions, format_report, gpu_state, h2t,  # noqa: E402
                            lib_cfg, oracle_decisions, rtol_for, snapshot)


class _AccView:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f2", "data": (ptr, False), "version": 3}


def main():
    family = sys.argv[1] if len(sys.argv) > 1 else "exact"
    updates = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    impl = sys.argv[3] if len(sys.argv) > 3 else "auto"
    use_graph = len(sys.argv) > 4 and sys.argv[4] == "graph"
    sharded = len(sys.argv) > 4 and sys.argv[4] in ("sharded", "sharded_graph")
    shard_graph = len(sys.argv) > 4 and sys.argv[4] == "sharded_graph"   # the launch bench.py times at W > 1
    many = len(sys.argv) > 4 and sys.argv[4] == "many"
    external = len(sys.argv) > 4 and sys.argv[4] == "external"
    acc32 = len(sys.argv) > 4 and sys.argv[4] == "acc32"      # SURVEY Z1 knob: fp32 accumulator, rn16, fp16 AR
    split = len(sys.argv) > 4 and sys.argv[4] == "split"      # smpu_config.split_tensors: buckets cut tensors
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = 3
    tensors = [("w0", 300_001, 0), ("b0", 1025, 1), ("w1", 262_144, 0), ("e", 131_072, 2), ("b1", 7, 1)]
    # u=3: finite A_r, overflow only after the sum (early decision undecided -> sweep -> skip);
    # u=4: finite 40000 after the sum (undecided -> sweep -> late apply); u=5, 6: non-finite A_r (early skip)
    inj = [dict(u=3, kind="RED_OVF", i=262_150), dict(u=4, kind="BIG", i=300_500),
           dict(u=5, kind="INF", r=world - 1, k=2, i=17), dict(u=6, kind="ACC_OVF", r=0, i=400_000)]
    wl = models.Workload("multi", tensors, world, c, injections=inj, family=family)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    obj = [P.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    # bucket threshold chosen so buckets split the vector at unaligned boundaries
    ar = {"auto": P.smpu.AR_AUTO, "nccl": P.smpu.AR_NCCL, "fused": P.smpu.AR_FUSED, "ce": P.smpu.AR_FUSED,
          "ce2": P.smpu.AR_FUSED}[impl]
    ocfg = O.Config(accum_fp32=acc32)
    step = P.UpdateStep(wl.numel, theta0 if rank == 0 else np.zeros_like(theta0),
                        lib_cfg(wl, ocfg, bucket_bytes=400_000, allreduce=ar, split_tensors=int(split),
                                ar_copy_engine={"ce": 1, "ce2": 2}.get(impl, 0)), world=world,
                        rank=rank,
                        nccl_id=obj[0], device=local)
    assert step.n_buckets >= 2
    fused = step.allreduce_impl == P.smpu.AR_FUSED
    if impl in ("fused", "ce", "ce2"):
        assert fused
    shard_step = None
    if sharded:   # the SURVEY f2 variant beside the replicated ctx, same inputs: must agree bitwise on its shard
        obj2 = [P.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj2, src=0)
        shard_step = P.UpdateStep(wl.numel, theta0 if rank == 0 else np.zeros_like(theta0),
                                  lib_cfg(wl, bucket_bytes=400_000, allreduce=P.smpu.AR_FUSED, sharded=1),
                                  world=world, rank=rank, nccl_id=obj2[0], device=local)
        ranges = shard_step.shard_ranges()
        assert sum(h - l for l, h in ranges) < lay.n
        cover = [None] * world
        dist.all_gather_object(cover, ranges)
        mark = np.zeros(lay.n, np.int32)
        for rr in cover:
            for l, h in rr:
                mark[l:h] += 1
        assert (mark == 1).all(), "shards must partition the vector"
        if shard_graph:
            sgbufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(c)]
            shard_step.graph_capture(sgbufs)
    orc = O.Oracle(theta0, ocfg) if rank == 0 else None
    mags = Magnitudes(theta0) if rank == 0 else None
    e = 7
    failures = []
    report = []
    if use_graph:
        gbufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(c)]
        if not fused:      # documented limitation: graphs at W > 1 need the fused all-reduce
            try:
                step.graph_capture(gbufs)
                failures.append("graph capture with the NCCL all-reduce should be refused")
            except P.SmpuError as ex:
                assert ex.status == P.smpu.EINVAL
            use_graph = False
        else:
            step.graph_capture(gbufs)
    for u in range(1, updates + 1):
        mine = [synth.micro_grad_cpu(wl, lay, u, rank, k, e) for k in range(1, c + 1)]
        toks = [synth.ntokens(wl, u, rank, k) for k in range(1, c + 1)]
        if use_graph:
            for k in range(c):
                gbufs[k].copy_(torch.from_numpy(mine[k].view(np.int16)))
            step.graph_launch(toks)
            res = step.result(u)
        elif external:     # the producer accumulates in place (torch fp16 copy/add), declares with None
            acc = torch.as_tensor(_AccView(step.accumulator_ptr(), lay.n), device="cuda")
            for k in range(c):
                g = h2t(mine[k]).view(torch.float16)
                acc.copy_(g) if k == 0 else acc.add_(g)
                step.accumulate(None, toks[k])
            res = step.step()
        elif many:     # resident micro-batches: the first one alone, then the rest (incl. the final) in one pass
            step.accumulate(h2t(mine[0]), toks[0])
            step.accumulate_many([h2t(x) for x in mine[1:]], toks[1:])
            res = step.step()
        else:
            for k in range(c):
                step.accumulate(h2t(mine[k]), toks[k])
            res = step.step()
        if shard_step is not None:
            if shard_graph:
                for k in range(c):
                    sgbufs[k].copy_(torch.from_numpy(mine[k].view(np.int16)))
                shard_step.graph_launch(toks)
                rs = shard_step.result(u)
            else:
                for k in range(c):
                    shard_step.accumulate(h2t(mine[k]), toks[k])
                rs = shard_step.step()
            if decisions(rs) != decisions(res):
                failures.append(f"update {u}: sharded decisions {decisions(rs)} vs replicated {decisions(res)}")
            if not np.array_equal(shard_step.get_state(P.smpu.STATE_W16), step.get_state(P.smpu.STATE_W16)):
                failures.append(f"update {u}: sharded w16 differs from replicated")
            for which in (P.smpu.STATE_MASTER, P.smpu.STATE_M, P.smpu.STATE_V):
                a_, b_ = shard_step.get_state(which), step.get_state(which)
                if not all(np.array_equal(a_[l:h], b_[l:h]) for l, h in ranges):
                    bad = [(l + int(j), float(a_[l + j]), float(b_[l + j])) for l, h in ranges
                           for j in np.nonzero(a_[l:h] != b_[l:h])[0][:3]]
                    failures.append(f"update {u}: sharded state {which} differs on this rank's shard: "
                                    f"{sum(int((a_[l:h] != b_[l:h]).sum()) for l, h in ranges)} elements, e.g. {bad[:4]}")
        R = step.get_state(P.smpu.STATE_ACCUM)
        st = gpu_state(step)
        h = hashlib.sha256(b"".join(st[x].tobytes() for x in ("theta", "m", "v", "w16"))).hexdigest()
        hs = [None] * world
        dist.all_gather_object(hs, (h, decisions(res)))
        if len({x[0] for x in hs}) != 1 or len({x[1] for x in hs}) != 1:
            failures.append(f"update {u}: replicas differ {hs}")
        if rank == 0:
            grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, e) for k in range(1, c + 1)] for r in range(world)]
            ntok = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(world)]
            before = snapshot(orc)
            ores = orc.update(grads, ntok)
            if ores["applied"]:
                mags.update(ores["R"], ores["e_used"], ores["N"], before["theta"], orc.theta, m_before=before["m"])
            # bitwise: exactly-summable values (any order), two operands (a + b == b + a), or the fused
            # all-reduce, which sums in the oracle's ascending rank order
            if family == "exact" or world == 2 or fused:
                if decisions(res) != oracle_decisions(ores):
                    failures.append(f"update {u}: decisions {decisions(res)} vs {oracle_decisions(ores)}")
                nan = np.isnan(ores["R"].view(np.float16))
                if not (np.array_equal(np.isnan(R.view(np.float16)), nan) and np.array_equal(R[~nan], ores["R"][~nan])):
                    failures.append(f"update {u}: reduced gradient differs")
                try:
                    check_state(st, snapshot(orc), mags, rtol_for(orc.s.t), where=f"update {u}", report=report)
                except AssertionError as ex:
                    failures.append(str(ex))
            else:
                # G_real, W > 2: NCCL's fp16 order is not pinned (reading R3, parity unpinned): report R's ulp distance
                # (informational) and check the decisions, which the bounded generator makes order-independent
                from tests.gpu_util import ulp16_dist
                fin = ~np.isnan(ores["R"].view(np.float16)) & ~np.isinf(ores["R"].view(np.float16))
                d = ulp16_dist(R[fin], ores["R"][fin])
                print(f"[rank0] update {u}: G_real R vs ascending-order oracle: max {d.max()} ulp, "
                      f"{(d > 0).mean():.2e} of elements differ", flush=True)
                if decisions(res)[:4] != oracle_decisions(ores)[:4]:
                    failures.append(f"update {u}: decisions {decisions(res)} vs {oracle_decisions(ores)}")
        e = res["scale_log2_next"]
    flags = [None] * world
    dist.all_gather_object(flags, failures)
    if shard_step is not None:
        shard_step.close()
    step.close()
    dist.destroy_process_group()
    allf = [f for fl in flags for f in fl]
    if allf:
        print("FAIL", *allf, sep="\n")
        sys.exit(1)
    if rank == 0:
        if report:
            print("errors:", format_report(report))
        print(f"multi-GPU parity ok: world={world} family={family} updates={updates} impl={impl} "
              f"(ran {'fused' if fused else 'nccl'}){' as CUDA graph' if use_graph else ''}"
              f"{' + sharded optimizer bitwise' if sharded else ''}{' (sharded ctx as CUDA graph)' if shard_graph else ''}{' via accumulate_many' if many else ''}"
              f"{' with in-place producer accumulation' if external else ''}{' with the fp32 accumulator' if acc32 else ''}{' with split-tensor buckets' if split else ''}")


if __name__ == "__main__":
    main()
