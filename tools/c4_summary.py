"""Summarise tools/c4_sweep.py JSONL files as one table per world size and update_freq.

usage: python tools/c4_summary.py OUT.txt FILE.jsonl [FILE.jsonl ...]
"""
import json
import sys


def main():
    out, files = sys.argv[1], sys.argv[2:]
    rows = []
    for f in files:
        for line in open(f):
            d = json.loads(line)
            d["_file"] = f
            rows.append(d)
    keys = sorted({(d["world"], d["update_freq"]) for d in rows}, key=lambda k: (k[0], -k[1]))
    lines = ["# C4 bucket sweep (SURVEY 8(d.1)): Transformer-big En-De, library-only update step (M1), G_real, CUDA graph,",
             "# replicated layout; exposed = T(W ranks) - T(same per-GPU work through a world = 1 ctx, same GPU, same run);",
             "# comm = the bucket all-reduce launches' own time (CUDA events); bus = 2 (W-1)/W x 2n B / comm (in situ).",
             ""]
    for w, c in keys:
        lines.append(f"## W = {w}, update_freq = {c}")
        lines.append(f"{'MiB':>6} {'pieces':>6} {'ce':>3} {'shape':>10} {'buckets':>7} {'T_ms':>7} {'T1_ms':>7} {'exposed_ms':>10} "
                     f"{'exp/T':>6} {'comm_ms':>8} {'exp/comm':>8} {'bus_GB/s':>8}  file")
        sel = [d for d in rows if d["world"] == w and d["update_freq"] == c]
        sel.sort(key=lambda d: (d["bucket_mib"], d.get("ar_pieces", 1), d.get("ar_copy_engine", 0),
                                d.get("ar_shape", "")))
        for d in sel:
            lines.append(f"{d['bucket_mib']:>6.0f} {d.get('ar_pieces', d.get('ar_tail_split', 1)):>6} "
                         f"{d.get('ar_copy_engine', 0):>3} {d.get('ar_shape', '148x256x1'):>10} {d['n_buckets']:>7} {d['T_update_ms']:>7.3f} "
                         f"{d['T_world1_ms']:>7.3f} {d['exposed_ms']:>10.3f} {d['exposed_frac_of_update']:>6.1%} "
                         f"{d['comm_ms']:>8.3f} {d['exposed_frac_of_comm']:>8.1%} {d['bus_gbs_in_situ']:>8.0f}  "
                         f"{d['_file']}")
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
