"""BASELINE.json configs[3] on W GPUs: Transformer-big En-Fr (221.9M params), update_freq 16, 5,200 updates with a
burst of four injected overflows (INF, NAN, ACC_OVF, RED_OVF) at u = 2500-2503 and 5000-5003.

Launched by tests/test_gpu_multi.py under torch.distributed.run.  Every rank generates its own exactly-summable
micro-gradients on its GPU at the current loss scale; rank 0 runs the oracle on sampled indices over all W ranks'
inputs.  Checked: decisions bitwise every update, the hand-derived scaler checkpoints (tests/golden/
scaler_trace_c3.txt), sampled theta/m/v/w16 after the run, bitwise-identical replicas.
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
from tests.conftest import golden  # noqa: E402
from tests.gpu_util import (RTOL_100, Magnitudes, check_state, decisions, gpu_state, lib_cfg,  # noqa: E402
                            oracle_decisions, snapshot)


def main():
    updates = int(sys.argv[1]) if len(sys.argv) > 1 else 5200
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = models.big_enfr(world=world)
    lay = synth.Layout(wl)
    c = wl.update_freq
    theta0 = torch.empty(lay.n, dtype=torch.float32, device="cuda")
    synth.theta0_gpu(theta0, wl)
    obj = [P.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    step = P.UpdateStep(wl.numel, theta0, lib_cfg(wl), world=world, rank=rank, nccl_id=obj[0], device=local)
    bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(c)]
    inj_u = {inj["u"] for inj in wl.injections}
    failures = []
    if rank == 0:
        idx = np.unique(np.concatenate([np.random.default_rng(3).integers(0, lay.n, 2048), lay.begin[1:-1],
                                        step.bucket_begin[1:-1], [inj["i"] for inj in wl.injections]]))
        orc = O.Oracle(synth.theta0_sample(wl, idx))
        mags = Magnitudes(orc.theta.copy())
        checks = {int(r[0]): tuple(map(int, r[1:])) for r in golden("scaler_trace_c3.txt")}
    e = 7
    for u in range(1, updates + 1):
        for k in range(1, c + 1):
            synth.micro_grad_gpu(bufs[k - 1], wl, lay, u, rank, k, e)
        toks = [synth.ntokens(wl, u, rank, k) for k in range(1, c + 1)]
        for k in range(c):
            step.accumulate(bufs[k], toks[k])
        res = step.step()
        if rank == 0:
            grads = [[synth.micro_grad_sample(wl, lay, idx, u, r, k, e) for k in range(1, c + 1)] for r in range(world)]
            ntok = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(world)]
            before = orc.theta.copy()
            ores = orc.update(grads, ntok, overflow=(u in inj_u))   # the bounded generator cannot overflow alone
            if ores["applied"]:
                mags.update(ores["R"], ores["e_used"], ores["N"], before, orc.theta)
            if decisions(res) != oracle_decisions(ores):
                failures.append(f"update {u}: {decisions(res)} vs {oracle_decisions(ores)}")
            if u in checks and (orc.e, orc.s.clean, orc.s.t) != checks[u]:
                failures.append(f"update {u}: scaler {(orc.e, orc.s.clean, orc.s.t)} vs golden {checks[u]}")
        e = res["scale_log2_next"]
    st = gpu_state(step)
    h = hashlib.sha256(b"".join(st[x].tobytes() for x in ("theta", "m", "v", "w16"))).hexdigest()
    hs = [None] * world
    dist.all_gather_object(hs, h)
    if len(set(hs)) != 1:
        failures.append(f"replicas differ: {hs}")
    if rank == 0:
        try:
            check_state({k2: v[idx] for k2, v in st.items()}, snapshot(orc), mags, RTOL_100, where="end of run")
        except AssertionError as ex:
            failures.append(str(ex))
        s = step.scalars()
        if updates == 5200 and (s["e"], s["clean"], s["t"], s["attempts"]) != (1, 197, 5192, 5200):
            failures.append(f"final scalars {s}")
    fl = [None] * world
    dist.all_gather_object(fl, failures)
    impl = step.allreduce_impl
    step.close()
    dist.destroy_process_group()
    allf = [f for x in fl for f in x]
    if allf:
        print("FAIL", *allf, sep="\n")
        sys.exit(1)
    if rank == 0:
        print(f"C3 ok: world={world} updates={updates} impl={impl}")


if __name__ == "__main__":
    main()
