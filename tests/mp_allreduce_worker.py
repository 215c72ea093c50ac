"""smpu_allreduce_accumulator at W ranks (collective primitive): every rank's accumulator holds its own G_real
vector; after the call every rank holds the oracle's ascending-rank fp16 sum (fused implementation: bitwise for
any values; NCCL implementation: bitwise only for W = 2)."""
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
from tests.gpu_util import lib_cfg  # noqa: E402


class _View:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}


def main():
    impl = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = models.Workload("ar", [("w0", 700_001, 0), ("b", 33, 1), ("e", 300_000, 2)], world, 1)
    lay = synth.Layout(wl)
    obj = [P.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ar = {"fused": P.smpu.AR_FUSED, "nccl": P.smpu.AR_NCCL}[impl]
    step = P.UpdateStep(wl.numel, synth.theta0_cpu(wl, lay), lib_cfg(wl, bucket_bytes=500_000, allreduce=ar),
                        world=world, rank=rank, nccl_id=obj[0], device=local)
    acc = torch.as_tensor(_View(step.accumulator_ptr(), lay.n), device="cuda")
    mine = [synth.micro_grad_cpu(wl, lay, 1, r, 1, 7) for r in range(world)]
    acc.copy_(torch.from_numpy(mine[rank].view(np.int16)))
    step.allreduce_accumulator()
    torch.cuda.synchronize()
    got = step.get_state(P.smpu.STATE_ACCUM)
    ok = True
    if impl == "fused" or world == 2:
        ok = np.array_equal(got, O.reduce(mine))
    hs = [None] * world
    dist.all_gather_object(hs, (ok, hashlib.sha256(got.tobytes()).hexdigest()))
    step.close()
    dist.destroy_process_group()
    if not all(h[0] for h in hs) or len({h[1] for h in hs}) != 1:
        print("FAIL", hs)
        sys.exit(1)
    if rank == 0:
        print(f"allreduce_accumulator ok: world={world} impl={impl}")


if __name__ == "__main__":
    main()
