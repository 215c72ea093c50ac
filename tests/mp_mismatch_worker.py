"""Ranks that disagree on a collective-shaping config field fail smpu_init with EINVAL on EVERY rank -- none hangs in
window registration or an LSA barrier (include/smpu.h, smpu_config.ar_*).  Then a consistent
init on the same process group succeeds and runs an update."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1806_00187_b200 as P  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    numel = [100_003, 4097]
    theta0 = np.zeros(sum(numel), np.float32)
    fails = []
    cases = [dict(ar_ctas=64 + rank), dict(ar_threads=256 if rank == 0 else 512), dict(update_freq=2 + rank),
             dict(bucket_bytes=(1 << 20) + rank), dict(sharded=rank % 2), dict(ar_copy_engine=rank % 2),
             dict(ar_pieces=1 + rank)]
    for kw in cases:
        obj = [P.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        try:
            st = P.UpdateStep(numel, theta0, P.config_default(**kw), world=world, rank=rank, nccl_id=obj[0],
                              device=local)
            st.close()
            fails.append(f"{kw}: init succeeded on rank {rank}")
        except P.SmpuError as ex:
            if ex.status != P.smpu.EINVAL or "disagree" not in str(ex):
                fails.append(f"{kw}: rank {rank} got {ex}")
    obj = [P.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    st = P.UpdateStep(numel, theta0, P.config_default(update_freq=1, ar_ctas=32, ar_copy_engine=1), world=world,
                      rank=rank, nccl_id=obj[0], device=local)
    g = torch.ones(sum(numel), dtype=torch.float16, device="cuda").view(torch.int16)
    st.accumulate(g, 10)
    r = st.step()
    if r["applied"] != 1 or r["ntokens_total"] != 10 * world:
        fails.append(f"consistent init: {r}")
    st.close()
    allf = [None] * world
    dist.all_gather_object(allf, fails)
    dist.destroy_process_group()
    flat = [f for x in allf for f in x]
    if flat:
        print("FAIL", *flat, sep="\n")
        sys.exit(1)
    if rank == 0:
        print(f"mismatch ok: {len(cases)} mismatched configs refused with EINVAL on all {world} ranks")


if __name__ == "__main__":
    main()
