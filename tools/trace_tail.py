"""Print the last update of a `bench.py --trace` timeline (one JSONL file per rank): every launch of the update
with its stream, start and end relative to the end of the update's last K1 (the moment the last micro-batch is
accumulated, after which only the exchange and Adam remain), plus per-stream busy time in that tail.

usage: python tools/trace_tail.py TRACE.N.rank0 [TRACE.N.rank1 ...]
"""
import collections
import json
import sys


def main():
    for path in sys.argv[1:]:
        ev = [json.loads(l) for l in open(path)]
        ev.sort(key=lambda e: e["start_ms"])
        # updates start at a k1_first launch
        starts = [i for i, e in enumerate(ev) if e["kernel"] == "k1_first"]
        upd = ev[starts[-1]:]
        k1 = [e for e in upd if e["kernel"] in ("k1_first", "k1_add", "k1_many")]
        t0 = max(e["end_ms"] for e in k1)
        t_first = upd[0]["start_ms"]
        t_end = max(e["end_ms"] for e in upd)
        print(f"== {path}: update {t_end - t_first:.3f} ms, tail after the last K1 {t_end - t0:.3f} ms")
        busy = collections.defaultdict(float)
        for e in upd:
            if e["end_ms"] <= t0 - 0.3:
                continue
            a, b = e["start_ms"] - t0, e["end_ms"] - t0
            busy[e["stream"]] += max(0.0, b - max(a, 0.0))
            print(f"  {e['stream']:>8} {e['kernel']:>12} {a:8.3f} {b:8.3f}  ({b - a:.3f})")
        print("  busy in the tail:", {k: round(v, 3) for k, v in busy.items()})


if __name__ == "__main__":
    main()
