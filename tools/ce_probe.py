"""Copy-engine (CE) peer bandwidth probe over NVLink, one process, all visible GPUs.

Measures what cudaMemcpyPeerAsync (torch cross-device copy_) moves between B200s: one direction, both directions at
once, several streams per direction, the W-rank push pattern (every GPU to every other GPU at once), and the same
push while an HBM-bound kernel runs on every GPU (does CE traffic slow the kernel, and the kernel the CE?).
CUDA events on the copy streams, best of R repetitions.  Output: one JSON object per line.
"""
import json
import sys

import torch


def ev(dev):
    return torch.cuda.Event(enable_timing=True)


def timed(fn, devs, reps=5):
    best = 1e30
    for _ in range(reps):
        for d in devs:
            torch.cuda.synchronize(d)
        starts, ends = {}, {}
        # one start / end event per device on its own default stream; fn enqueues on side streams that wait on them
        for d in devs:
            with torch.cuda.device(d):
                starts[d] = torch.cuda.Event(enable_timing=True)
                starts[d].record()
        fn(starts)
        for d in devs:
            with torch.cuda.device(d):
                ends[d] = torch.cuda.Event(enable_timing=True)
                ends[d].record()
        for d in devs:
            torch.cuda.synchronize(d)
        ms = max(starts[d].elapsed_time(ends[d]) for d in devs)
        best = min(best, ms)
    return best


def main():
    n = torch.cuda.device_count()
    MB = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    nbytes = MB << 20
    devs = list(range(n))
    for a in devs:
        for b in devs:
            if a != b:
                assert torch.cuda.can_device_access_peer(a, b)
    src = {d: torch.empty(nbytes, dtype=torch.uint8, device=d).fill_(d + 1) for d in devs}
    dst = {d: {p: torch.empty(nbytes, dtype=torch.uint8, device=d) for p in devs if p != d} for d in devs}
    streams = {d: [torch.cuda.Stream(device=d) for _ in range(8)] for d in devs}

    def push(pairs, split):
        def fn(starts):
            # each (a -> b) copy issued on a's streams (the source GPU's CEs drive the write over NVLink)
            used = {}
            for (a, b) in pairs:
                chunk = nbytes // split
                for s in range(split):
                    k = used.get(a, 0)
                    used[a] = k + 1
                    st = streams[a][k % len(streams[a])]
                    st.wait_event(starts[a])
                    with torch.cuda.stream(st):
                        dst[b][a][s * chunk:(s + 1) * chunk].copy_(src[a][s * chunk:(s + 1) * chunk], non_blocking=True)
            for a in set(x for x, _ in pairs):
                cur = torch.cuda.current_stream(a)
                for st in streams[a]:
                    cur.wait_stream(st)
        return fn

    def report(name, pairs, split, extra=None):
        ms = timed(push(pairs, split), devs)
        per_src = {}
        for a, _ in pairs:
            per_src[a] = per_src.get(a, 0) + nbytes
        out_gbs = max(per_src.values()) / (ms * 1e-3) / 1e9
        row = {"probe": name, "mib": MB, "split": split, "ms": ms, "out_gbs_per_gpu": out_gbs,
               "pairs": len(pairs)}
        if extra:
            row.update(extra)
        print(json.dumps(row), flush=True)
        return ms

    report("uni 0->1", [(0, 1)], 1)
    report("uni 0->1", [(0, 1)], 4)
    report("bidir 0<->1", [(0, 1), (1, 0)], 1)
    report("bidir 0<->1", [(0, 1), (1, 0)], 4)
    allpairs = [(a, b) for a in devs for b in devs if a != b]
    for split in (1, 2, 4):
        report(f"push all-to-all W={n}", allpairs, split)

    # rotating partners, one stream per GPU: in round j GPU a sends to a + 1 + j (a perfect matching per round)
    def rotate(starts):
        for a in devs:
            st = streams[a][0]
            st.wait_event(starts[a])
            with torch.cuda.stream(st):
                for j in range(n - 1):
                    b = (a + 1 + j) % n
                    dst[b][a].copy_(src[a], non_blocking=True)
            torch.cuda.current_stream(a).wait_stream(st)
    ms = timed(rotate, devs)
    print(json.dumps({"probe": f"push rotating partners W={n}", "mib": MB, "ms": ms,
                      "out_gbs_per_gpu": (n - 1) * nbytes / (ms * 1e-3) / 1e9}), flush=True)

    # the same all-to-all push while an HBM-bound copy runs on every GPU (the in-situ question)
    big = {d: torch.empty(1 << 30, dtype=torch.uint8, device=d) for d in devs}
    big2 = {d: torch.empty(1 << 30, dtype=torch.uint8, device=d) for d in devs}
    hbm_alone = timed(lambda s: [big2[d].copy_(big[d]) for d in devs], devs)

    hs = {d: torch.cuda.Stream(device=d) for d in devs}

    def both(starts):
        for d in devs:
            hs[d].wait_event(starts[d])
            with torch.cuda.stream(hs[d]):
                big2[d].copy_(big[d])
        push(allpairs, 2)(starts)
        for d in devs:
            torch.cuda.current_stream(d).wait_stream(hs[d])
    ms_push_alone = timed(push(allpairs, 2), devs)
    ms_both = timed(both, devs)
    print(json.dumps({"probe": f"in situ W={n}", "hbm_copy_alone_ms": hbm_alone,
                      "hbm_copy_gbs": 2 * (1 << 30) / (hbm_alone * 1e-3) / 1e9,
                      "push_alone_ms": ms_push_alone, "both_ms": ms_both,
                      "serial_sum_ms": hbm_alone + ms_push_alone}), flush=True)


if __name__ == "__main__":
    main()
