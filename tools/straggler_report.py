#!/usr/bin/env python
"""Straggler analysis on a synthetic WMT-sized corpus with libsmpu_sched.so (PAPER.md 5).

Corpus: 4.5M sentence pairs, log-normal lengths (median 24), target/source ratio in [0.67, 1.5].
'True' sub-batch cost (stands in for the real model's forward+backward, which is out of scope): padded tokens
plus an attention-like quadratic term, t = 1.35 us * S * (Ls + Lt) / 2 + 2 ns * S * (Ls^2 + Lt^2) + 0.2 ms.
The timing table is fitted on 2,000 noisy measurements; time-balanced sub-batches target the 90th
percentile.  Idle fractions for W = 8 workers (one DGX-1 / one 8-GPU box), update_freq 1 and 16.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1806_00187_b200 import sched as S  # noqa: E402


def true_cost(src, tgt, order, begin):
    out = np.empty(len(begin) - 1)
    for b in range(len(begin) - 1):
        ids = order[begin[b]:begin[b + 1]]
        s, ls, lt = len(ids), src[ids].max(), tgt[ids].max()
        out[b] = 1.35e-6 * s * (ls + lt) / 2 + 2e-9 * s * (ls * ls + lt * lt) + 2e-4
    return out


def main():
    rng = np.random.default_rng(0)
    n = 4_500_000
    src = np.clip(np.round(rng.lognormal(np.log(24), 0.6, n)), 1, 250).astype(np.int32)
    tgt = np.clip(np.round(src * rng.uniform(0.67, 1.5, n)), 1, 250).astype(np.int32)
    o1, b1 = S.token_budget(src, tgt, 3500)
    t1 = true_cost(src, tgt, o1, b1)
    # timing table from noisy measurements of a random 2,000 token-budget sub-batches
    pick = rng.choice(len(b1) - 1, 2000, replace=False)
    sent = np.array([b1[b + 1] - b1[b] for b in pick])
    ms = np.array([src[o1[b1[b]:b1[b + 1]]].max() for b in pick])
    mt = np.array([tgt[o1[b1[b]:b1[b + 1]]].max() for b in pick])
    meas = t1[pick] * rng.normal(1.0, 0.03, pick.size)
    coef = S.fit_timing(sent, ms, mt, meas)
    target = np.percentile(S.estimate(src, tgt, o1, b1, coef), 90)
    o2, b2 = S.time_balanced(src, tgt, coef, target)
    t2 = true_cost(src, tgt, o2, b2)
    tok = lambda o, b: np.array([tgt[o[b[i]:b[i + 1]]].sum() for i in range(len(b) - 1)])  # noqa: E731
    lines = [__doc__.strip(), "",
             f"token-budget 3.5k: {len(b1) - 1} sub-batches, time mean {t1.mean()*1e3:.1f} ms, "
             f"min/mean {t1.min()/t1.mean():.2f}, max/mean {t1.max()/t1.mean():.2f} "
             f"(paper Fig. 6: 0.049/0.11 = 0.45, 0.228/0.11 = 2.07), CV {t1.std()/t1.mean():.3f}",
             f"fitted timing model a={coef[0]:.3e} b={coef[1]:.3e} c={coef[2]:.3e}; 90th-percentile target "
             f"{target*1e3:.1f} ms",
             f"time-balanced: {len(b2) - 1} sub-batches, time mean {t2.mean()*1e3:.1f} ms, CV {t2.std()/t2.mean():.3f}"]
    for name, o, b, t in (("token-budget", o1, b1, t1), ("time-balanced", o2, b2, t2)):
        perm = rng.permutation(len(t))
        tt, kk = t[perm], tok(o, b)[perm]
        for c in (1, 16):
            r = S.simulate(tt, 8, c)
            used = r["steps"] * 8 * c
            lines.append(f"{name:14s} W=8 update_freq={c:2d}: idle fraction {r['idle_fraction']:.3f}, "
                         f"throughput {kk[:used].sum() / r['wall'] / 1e3:.1f}k target tokens/s (compute only)")
    text = "\n".join(lines) + "\n"
    print(text)
    with open(os.path.join(ROOT, "profiles", "r1_straggler.txt"), "w") as f:
        f.write(text)


if __name__ == "__main__":
    main()
