#!/usr/bin/env python
"""Per-config CPU oracle timings ("CPU oracle, timed beside it"): whole oracle updates of

    C0  tiny, W = 1, c = 2, all 10 updates (its injected inf at u = 5 included)
    C1  Transformer-base En-De, W = 1, c = 1, 3 updates
    C2  Transformer-big En-De, W = 1, c = 16, 1 update
    C2' Transformer-big En-De, W = 8 ranks emulated in-process, c = 16, 1 update

at 1 thread and at `nproc` threads (OpenMP over elements), with the host CPU model.  The oracle runs as it stands
(oracle.Oracle.update); full vectors that do not fit the host comfortably are processed as consecutive index
chunks, each a whole oracle update of its slice (every stage but the decision is elementwise and the G_real inputs
never overflow, so the chunks together do exactly one full update's work).  Only Oracle.update is timed; the input
generation is not.  1-thread runs of the W = 8 config time a 1/8 slice and say so.

    python tools/oracle_timings.py [--out profiles/r2_oracle_timings.txt] [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402
from synth import models  # noqa: E402


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def timed_updates(wl, updates, frac=1.0, chunk=1 << 23):
    """Seconds of Oracle.update work for `updates` whole updates over the first frac of the vector, chunked."""
    lay = synth.Layout(wl)
    n = int(lay.n * frac)
    W, c = wl.world, wl.update_freq
    total = 0.0
    orcs = []
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        th = synth.theta0_sample(wl, np.arange(lo, hi, dtype=np.int64)) if lay.n > chunk else \
            synth.theta0_cpu(wl, lay)[lo:hi]
        orcs.append((lo, hi, O.Oracle(th)))
    decisions = []
    for u in range(1, updates + 1):
        ov_any = False
        for lo, hi, orc in orcs:
            e = orc.e
            grads = [[synth.micro_grad_range(wl, lay, lo, hi, u, r, k, e) for k in range(1, c + 1)] for r in range(W)]
            toks = [[synth.ntokens(wl, u, r, k) for k in range(1, c + 1)] for r in range(W)]
            t0 = time.perf_counter()
            res = orc.update(grads, toks)
            total += time.perf_counter() - t0
            ov_any |= bool(res["overflow"])
        decisions.append(int(ov_any))
    return total, n, decisions


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_oracle_timings.txt"))
    ap.add_argument("--quick", action="store_true", help="small fractions (a smoke run of the tool itself)")
    args = ap.parse_args()
    nproc = os.cpu_count() or 1
    q = 0.01 if args.quick else 1.0
    tiny = models.tiny()
    cases = [("C0 tiny W=1 c=2 (10 updates)", tiny, 10, 1.0),
             ("C1 base En-De W=1 c=1 (3 updates)", models.base_ende(), 3, q),
             ("C2 big En-De W=1 c=16 (1 update)", models.big_ende(1, 16), 1, q),
             ("C2' big En-De W=8 emulated c=16 (1 update)", models.big_ende(8, 16), 1, q)]
    rows = []
    for threads in (1, nproc):
        O.set_threads(threads)
        for name, wl, ups, frac in cases:
            if threads == 1 and wl.world == 8:
                frac = frac / 8          # 1 thread x 27G element-adds: time a 1/8 slice, say so
            secs, n, dec = timed_updates(wl, ups, frac)
            grad_elems = wl.world * wl.update_freq * n * ups
            row = {"config": name, "threads": threads, "updates": ups, "elements_timed": n, "n_params": wl.n,
                   "fraction_of_vector": n / wl.n, "oracle_seconds": secs,
                   "seconds_per_full_update": secs / ups * wl.n / n, "grad_elems_per_s": grad_elems / secs,
                   "overflow_decisions": dec}
            rows.append(row)
            print(json.dumps(row), flush=True)
    hdr = {"cpu_model": cpu_model(), "nproc": nproc, "tool": "tools/oracle_timings.py",
           "note": "Oracle.update only (inputs generated outside the timed region); chunked whole updates"}
    with open(args.out, "w") as f:
        f.write("# SURVEY 8(d.4) per-config CPU oracle timings on the GPU box's host cores\n")
        f.write(json.dumps(hdr) + "\n")
        f.write(f"{'config':46s} {'thr':>4s} {'frac':>6s} {'s/full update':>14s} {'grad elems/s':>13s}\n")
        for r in rows:
            f.write(f"{r['config']:46s} {r['threads']:4d} {r['fraction_of_vector']:6.3f} "
                    f"{r['seconds_per_full_update']:14.2f} {r['grad_elems_per_s']:13.3e}\n")
        for r in rows:
            f.write(json.dumps(r) + "\n")
    print("wrote", args.out)


if __name__ == "__main__":
    main()
