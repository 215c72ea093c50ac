"""World invariance on W GPUs ("(W=4, c=1) vs (W=1, c=4) ... identical"):
the same W micro-batches processed as (W ranks, update_freq 1) through the fused all-reduce, or as (1 rank,
update_freq W) on rank 0, give bitwise identical theta/m/v/w16 and decisions -- for G_real values, because the
fused all-reduce adds rank contributions in ascending order, the same association as local accumulation.
"""
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
from tests.gpu_util import decisions, h2t, lib_cfg  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tensors = [("w0", 300_001, 0), ("b0", 1025, 1), ("e", 131_072, 2), ("b1", 7, 1)]
    # micro-batch j of update u is synth (u, r=0, k=j+1) of the (W=1, c=W) numbering, on every layout
    wl1 = models.Workload("winv", tensors, 1, world,
                          injections=[dict(u=3, kind="INF", r=0, k=world, i=17)])
    lay = synth.Layout(wl1)
    theta0 = synth.theta0_cpu(wl1, lay)
    obj = [P.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    wlW = models.Workload("winv", tensors, world, 1)
    multi = P.UpdateStep(wl1.numel, theta0, lib_cfg(wlW, bucket_bytes=300_000, allreduce=P.smpu.AR_FUSED),
                         world=world, rank=rank, nccl_id=obj[0], device=local)
    # (1, c = W) twice: unfused, whose accumulator holds R like the multi-rank ctx's, and the default fused
    # last micro-batch (R consumed without being stored: compared on theta/m/v/w16)
    single = P.UpdateStep(wl1.numel, theta0, lib_cfg(wl1, bucket_bytes=300_000, fuse_final=0)) if rank == 0 else None
    fused = P.UpdateStep(wl1.numel, theta0, lib_cfg(wl1, bucket_bytes=300_000)) if rank == 0 else None
    failures = []
    e = 7
    for u in range(1, 7):
        micro = [synth.micro_grad_cpu(wl1, lay, u, 0, j, e) for j in range(1, world + 1)]
        toks = [synth.ntokens(wl1, u, 0, j) for j in range(1, world + 1)]
        multi.accumulate(h2t(micro[rank]), toks[rank])
        rm = multi.step()
        if rank == 0:
            for j in range(world):
                single.accumulate(h2t(micro[j]), toks[j])
                fused.accumulate(h2t(micro[j]), toks[j])
            rs, rf = single.step(), fused.step()
            if not decisions(rm) == decisions(rs) == decisions(rf):
                failures.append(f"update {u}: decisions {decisions(rm)} vs {decisions(rs)} vs {decisions(rf)}")
            for w in range(5):
                if not np.array_equal(multi.get_state(w), single.get_state(w)):
                    failures.append(f"update {u}: state {w} differs between (W={world}, c=1) and (1, c={world})")
                if w < 4 and not np.array_equal(multi.get_state(w), fused.get_state(w)):
                    failures.append(f"update {u}: state {w} differs between (W={world}, c=1) and fused (1, c={world})")
        e = rm["scale_log2_next"]
    fl = [None] * world
    dist.all_gather_object(fl, failures)
    if single is not None:
        single.close()
        fused.close()
    multi.close()
    dist.destroy_process_group()
    allf = [f for x in fl for f in x]
    if allf:
        print("FAIL", *allf[:10], sep="\n")
        sys.exit(1)
    if rank == 0:
        print(f"world invariance ok: (W={world}, c=1) == (W=1, c={world}) bitwise")


if __name__ == "__main__":
    main()
