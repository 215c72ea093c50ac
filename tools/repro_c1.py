"""Repro of the first W > 1 fuzz failure (r2t): W = 2, c = 1, an INF on rank 0 (u = 1, i = 1), tensors [1, 31], one
bucket per tensor -- the update applied although R held the INF (K1's max|A| statistic lost ragged-head values;
fixed).  Prints decisions, oracle decisions and R[1] for a few layouts."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import synth
from synth import models
import paper_1806_00187_b200 as P
from tests.gpu_util import lib_cfg, decisions, oracle_decisions, h2t


def run(tensors, W, c, bucket_bytes, inj, mode="calls"):
    wl = models.Workload("repro", tensors, W, c, injections=inj)
    lay = synth.Layout(wl)
    theta0 = synth.theta0_cpu(wl, lay)
    grp = P.VirtualGroup(wl.numel, theta0, lib_cfg(wl, bucket_bytes=bucket_bytes), world=W)
    ms = grp.members
    orc = O.Oracle(theta0)
    out = []
    for u in (1, 2):
        grads = [[synth.micro_grad_cpu(wl, lay, u, r, k, orc.e) for k in range(1, c + 1)] for r in range(W)]
        toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(W)]
        keep = []
        for k in range(c):
            for r in range(W):
                t = h2t(grads[r][k])
                keep.append(t)
                ms[r].accumulate(t, toks[r][k])
        torch.cuda.synchronize()
        accs = [m.get_state(P.smpu.STATE_ACCUM) for m in ms]
        for m in ms:
            m.step(wait=False)
        res = [m.result(u) for m in ms]
        ores = orc.update(grads, toks)
        out.append((u, [decisions(x)[:2] for x in res], oracle_decisions(ores)[:2],
                    [hex(int(a[1])) for a in accs], hex(int(grads[0][0][1]))))
    grp.close()
    return out


for args in [([("t0", 1, 0), ("t1", 31, 0)], 2, 1, 2), ([("t0", 1, 0), ("t1", 31, 0)], 2, 1, 1 << 20),
             ([("t0", 1, 0), ("t1", 31, 0)], 2, 2, 2), ([("t0", 100, 0), ("t1", 3100, 0)], 2, 1, 2),
             ([("t0", 1, 0), ("t1", 31, 0)], 3, 1, 2)]:
    inj = [dict(u=1, kind="INF", i=1, r=0, k=1)]
    print(args, run(*args, inj), flush=True)
