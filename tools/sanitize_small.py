"""Small W=1 run of every kernel path for compute-sanitizer (memcheck / racecheck): ragged tensors, unaligned
buckets, bucket-wise and whole micro-batches, accumulate_many, host (staged) inputs, graph replay, a skip."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1806_00187_b200 as P  # noqa: E402
import synth  # noqa: E402
from synth import models  # noqa: E402

tensors = [("a", 17, 1), ("b", 10_003, 0), ("c", 4_096, 2), ("d", 5, 1), ("e", 25_001, 0)]
wl = models.Workload("san", tensors, 1, 3, injections=[dict(u=2, kind="INF", r=0, k=3, i=10_010)])
lay = synth.Layout(wl)
cfg = P.config_default(update_freq=3, bucket_bytes=16 * 1024)
step = P.UpdateStep(wl.numel, synth.theta0_cpu(wl, lay), cfg)
bufs = [torch.empty(lay.n, dtype=torch.int16, device="cuda") for _ in range(3)]
for u in range(1, 5):
    g = [synth.micro_grad_cpu(wl, lay, u, 0, k, 7) for k in (1, 2, 3)]
    t = [100, 200, 300]
    dev = [torch.from_numpy(x.view(np.int16)).cuda() for x in g]
    if u == 1:
        for k in range(3):
            step.accumulate(dev[k], t[k])
    elif u == 2:
        step.accumulate(g[0], t[0])                       # pageable host input (staged H2D)
        step.accumulate_many(dev[1:2], t[1:2])
        step.micro_begin(t[2])
        bb = step.bucket_begin
        for b in reversed(range(step.n_buckets)):
            step.accumulate_bucket(b, dev[2][bb[b]:bb[b + 1]])
    else:
        step.accumulate_many(dev, t)
    print(u, step.step())
step.graph_capture(bufs)
for k in range(3):
    bufs[k].copy_(dev[k])
step.graph_launch([1, 2, 3])
print(step.result(5))
step.graph_capture(bufs, resident=True)
step.graph_launch([1, 2, 3])
print(step.result(6))
step.close()
print("sanitizer workload done")
