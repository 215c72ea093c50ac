#!/usr/bin/env python
"""Straggler analysis calibrated on the REAL model (PAPER.md 5) -- on a B200.

Round 1 ran libsmpu_sched.so on an invented cost model (tools/straggler_report.py).  Here every sub-batch time is a
measurement: the forward + backward of the paper's Transformer-big (producer/transformer.py, fp16, dropout 0.3,
label smoothing 0.1) on a sub-batch of S sentences padded to (Ls, Lt), timed with CUDA events (median of 3 after a
warm-up).

  1. Corpus: 4.5M sentence pairs, log-normal lengths (median 24 tokens, at most 250), target/source
     ratio in [0.67, 1.5] (P:278's filter).  Token-budget sub-batches of at most 3.5k tokens.
  2. Time a random sample of the token-budget sub-batches (--measure, default 240).  Their spread is the paper's
     Fig. 6 observation.
  3. Timing table: fit t = a S Ls + b S Lt + c (libsmpu_sched) on 2/3 of the measurements, report its error
     on the held-out third.
  4. Time-balanced sub-batches at the 90th-percentile target; time a random sample of those too.
  5. Idle fraction of synchronous SGD at W = 8, update_freq 1 and 16, simulated (smpu_sched_simulate)
     over streams of MEASURED sub-batch times drawn from each batching's sample.

    python tools/straggler_calibrate.py [--measure 240] [--out profiles/r2_straggler_measured.txt]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "producer"))

from paper_1806_00187_b200 import sched as S  # noqa: E402
from synth import models  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--measure", type=int, default=240)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_straggler_measured.txt"))
    ap.add_argument("--corpus", type=int, default=4_500_000)
    ap.add_argument("--eager", action="store_true", help="time the eager producer (launch-bound) instead of graphs")
    args = ap.parse_args()
    import torch
    from transformer import GraphedProducer, Producer, TransformerBig

    rng = np.random.default_rng(0)
    n = args.corpus
    src = np.clip(np.round(rng.lognormal(np.log(24), 0.6, n)), 1, 250).astype(np.int32)
    tgt = np.clip(np.round(src * rng.uniform(0.67, 1.5, n)), 1, 250).astype(np.int32)
    o1, b1 = S.token_budget(src, tgt, 3500)

    wl = models.big_ende()
    nparam = wl.n
    w16 = (torch.randn(nparam, device="cuda") * 0.02).to(torch.float16)
    model = TransformerBig(wl.tensors, w16, dropout=0.3, max_len=256)
    grad = torch.empty(nparam, dtype=torch.float16, device="cuda")
    prod = Producer(model, grad, torch.tensor([128.0], device="cuda"), seed=0)
    gp = None if args.eager else GraphedProducer(prod, [0] * len(wl.tensors), 1)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)

    def shape_of(order, begin, b):
        ids = order[begin[b]:begin[b + 1]]
        return len(ids), int(src[ids].max()), int(tgt[ids].max())

    def time_shape(s, ls, lt, reps=3):
        a = torch.randint(4, model.vocab, (s, ls), device="cuda", generator=gen)
        t = torch.randint(4, model.vocab, (s, lt + 1), device="cuda", generator=gen)
        run = prod.micro if gp is None else gp.micro
        run(a, t[:, :-1], t[:, 1:])                 # warm-up (allocator, kernel selection / graph capture)
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(a, t[:, :-1], t[:, 1:])
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e-3)
        if gp is not None:
            gp.forget()                             # one graph (and its activation pool) per shape at a time
        return float(np.median(out))

    def measure(order, begin, k):
        pick = rng.choice(len(begin) - 1, min(k, len(begin) - 1), replace=False)
        shp = [shape_of(order, begin, int(b)) for b in pick]
        sec = np.array([time_shape(*x) for x in shp])
        return np.array(shp, dtype=np.int64), sec

    shp1, t1 = measure(o1, b1, args.measure)
    fit = rng.permutation(len(t1))
    tr, te = fit[: 2 * len(t1) // 3], fit[2 * len(t1) // 3:]
    coef = S.fit_timing(shp1[tr, 0], shp1[tr, 1], shp1[tr, 2], t1[tr])
    pred = coef[0] * shp1[:, 0] * shp1[:, 1] + coef[1] * shp1[:, 0] * shp1[:, 2] + coef[2]
    err = np.abs(pred[te] - t1[te]) / t1[te]
    target = np.percentile(S.estimate(src, tgt, o1, b1, coef), 90)
    o2, b2 = S.time_balanced(src, tgt, coef, target)
    shp2, t2 = measure(o2, b2, args.measure)

    lines = [__doc__.strip().split("\n\n")[0], "",
             f"GPU: {torch.cuda.get_device_name()}; model Transformer-big En-De ({nparam} params), fp16 fwd+bwd, "
             f"{'eager PyTorch (launch-bound)' if gp is None else 'one CUDA graph per sub-batch shape'}",
             f"token-budget 3.5k: {len(b1) - 1} sub-batches (paper: 44K, P:319); measured {len(t1)}: "
             f"mean {t1.mean()*1e3:.2f} ms, min/mean {t1.min()/t1.mean():.2f}, max/mean {t1.max()/t1.mean():.2f} "
             f"(paper Fig. 6 on V100: 0.45 / 2.07), CV {t1.std()/t1.mean():.3f}",
             f"timing table t = a S Ls + b S Lt + c fitted on {len(tr)}: a={coef[0]:.3e} b={coef[1]:.3e} "
             f"c={coef[2]:.3e} s; held-out {len(te)}: median |err| {np.median(err)*100:.1f}%, "
             f"90th pct {np.percentile(err, 90)*100:.1f}%",
             f"90th-percentile target {target*1e3:.2f} ms -> time-balanced: {len(b2) - 1} sub-batches; measured "
             f"{len(t2)}: mean {t2.mean()*1e3:.2f} ms, CV {t2.std()/t2.mean():.3f}"]
    res = {"token_budget": {"sub_batches": len(b1) - 1, "measured": len(t1), "mean_ms": t1.mean() * 1e3,
                            "cv": t1.std() / t1.mean()},
           "time_balanced": {"sub_batches": len(b2) - 1, "measured": len(t2), "mean_ms": t2.mean() * 1e3,
                             "cv": t2.std() / t2.mean()},
           "coef": list(map(float, coef)), "heldout_median_rel_err": float(np.median(err))}
    for name, shp, t, nb in (("token-budget", shp1, t1, len(b1) - 1), ("time-balanced", shp2, t2, len(b2) - 1)):
        stream = t[rng.integers(0, len(t), nb)]            # a corpus-length stream of measured sub-batch times
        tok = (shp[:, 0] * shp[:, 2]).astype(np.float64)   # padded target tokens of each measured sub-batch
        for c in (1, 16):
            r = S.simulate(stream, 8, c)
            res[f"{name}_W8_c{c}_idle"] = r["idle_fraction"]
            lines.append(f"{name:14s} W=8 update_freq={c:2d}: idle fraction {r['idle_fraction']:.3f} "
                         f"(simulated over measured times; mean padded target tokens per sub-batch {tok.mean():.0f})")
    lines.append("")
    lines.append(json.dumps(res))
    text = "\n".join(lines) + "\n"
    print(text)
    with open(args.out, "w") as f:
        f.write(text)
        f.write("# measured sub-batches: sentences max_src max_tgt seconds (token-budget, then time-balanced)\n")
        for tag, shp, t in (("tb", shp1, t1), ("bal", shp2, t2)):
            for (s_, a_, b_), x in zip(shp, t):
                f.write(f"{tag} {s_} {a_} {b_} {x:.6f}\n")


if __name__ == "__main__":
    main()
