#!/usr/bin/env python
"""bucket-size sweep of the Transformer-big En-De update at W ranks (torchrun, one GPU per rank),
at update_freq 16 and 1, M1 (the library alone, inputs resident in HBM), the paper's replicated update.

For every threshold in {1, 2, 4, 8, 16, 32, 64, 128, 150, 256} MiB (whole-tensor buckets):
  T_update     CUDA-graph replay of one whole update (the bench's timed path), CUDA events, max over ranks
  exposed      T_update - T_world1, T_world1 = the same per-GPU work through a world = 1 ctx (fuse_final = 0) on
               the same GPU in the same run (no exchange)
  comm_ms      the bucket all-reduce kernels' summed device time per update (CUDA events, call-by-call region)
  bus GB/s     in situ, nccl-tests convention 2 (W-1)/W x 2n / comm_ms
and exposed / T_update (the "< 10%" headline, reading R25), exposed / comm_ms (the fraction of the communication
not hidden).

    torchrun --nproc-per-node W tools/c4_sweep.py [--c 16,1] [--mib 1,2,...] [--out profiles/r2_c4_sweep_wW.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c", default="16,1")
    ap.add_argument("--mib", default="1,2,4,8,16,32,64,128,150,256")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sharded", action="store_true", help="time the f2 layout instead of the replicated one")
    ap.add_argument("--out", default=None)
    ap.add_argument("--pieces", default="1", help="comma list of smpu_config.ar_pieces values to time")
    ap.add_argument("--ce", default="0", help="comma list of smpu_config.ar_copy_engine values to time")
    ap.add_argument("--shape", default="148x256x1",
                    help="comma list of all-reduce shapes CTAS x THREADS x UNROLL (smpu_config.ar_ctas/threads/unroll)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1806_00187_b200 as P
    import synth
    from synth import models
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    def mx(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def new_id():
        obj = [P.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def graph_ms(st, grads, toks, w):
        st.graph_capture(grads)
        for _ in range(args.warmup):
            st.graph_launch(toks, stream)
        torch.cuda.synchronize()
        if w > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            st.graph_launch(toks, stream)
        b.record(stream)
        torch.cuda.synchronize()
        if w > 1:
            dist.barrier()
        return a.elapsed_time(b) / args.steps

    def comm_ms(st, grads, toks):
        for _ in range(args.warmup):
            for k in range(len(grads)):
                st.accumulate(grads[k], toks[k], stream)
            st.step(stream, wait=False)
        torch.cuda.synchronize()
        dist.barrier()
        st.kernel_stats(reset=True)
        st.set_timing(True)
        for _ in range(args.steps):
            for k in range(len(grads)):
                st.accumulate(grads[k], toks[k], stream)
            st.step(stream, wait=False)
        torch.cuda.synchronize()
        dist.barrier()
        st.set_timing(False)
        s = st.kernel_stats(reset=True)
        return s["allreduce"]["ms"] / args.steps, s["allreduce"]["launches"] / args.steps

    out = []
    for c in [int(x) for x in args.c.split(",")]:
        wl = models.big_ende(world, c)
        lay = synth.Layout(wl)
        n = lay.n
        theta0 = torch.empty(n, dtype=torch.float32, device="cuda")
        synth.theta0_gpu(theta0, wl)
        grads = []
        for k in range(1, c + 1):
            g = torch.empty(n, dtype=torch.int16, device="cuda")
            synth.micro_grad_gpu(g, wl, lay, 1, rank, k, 7)
            grads.append(g)
        toks = [synth.ntokens(wl, 1, rank, k) for k in range(1, c + 1)]
        base_cfg = P.config_default(update_freq=c, fuse_final=0)
        base_cfg.growth_interval = 1 << 40
        s1 = P.UpdateStep(wl.numel, theta0, base_cfg, world=1, rank=0, device=local)
        t1 = mx(graph_ms(s1, grads, toks, 1))
        s1.close()
        for mib, split, ce, shape in [(float(x), int(y), int(z), sh) for x in args.mib.split(",")
                                      for y in args.pieces.split(",") for z in args.ce.split(",")
                                      for sh in args.shape.split(",")]:
            ctas, threads, unroll = (int(v) for v in shape.split("x"))
            cfg = P.config_default(update_freq=c, bucket_bytes=int(mib * (1 << 20)), sharded=int(args.sharded),
                                   ar_pieces=split, ar_copy_engine=ce, ar_ctas=ctas, ar_threads=threads,
                                   ar_unroll=unroll)
            cfg.growth_interval = 1 << 40
            t0 = time.perf_counter()
            st = P.UpdateStep(wl.numel, theta0, cfg, world=world, rank=rank, nccl_id=new_id(), device=local)
            init_s = time.perf_counter() - t0
            cm, launches = comm_ms(st, grads, toks)
            cm = mx(cm)
            T = mx(graph_ms(st, grads, toks, world))
            res = st.result(st.scalars()["attempts"])
            assert res["applied"] == 1, res
            phases = 1 if args.sharded else 2
            bus = phases * n * 2 * (world - 1) / world / (cm * 1e-3) / 1e9 if cm > 0 else None
            row = {"world": world, "update_freq": c, "bucket_mib": mib, "ar_pieces": split, "ar_copy_engine": ce, "ar_shape": shape,
                   "n_buckets": st.n_buckets,
                   "layout": "sharded" if args.sharded else "replicated", "T_update_ms": T, "T_world1_ms": t1,
                   "exposed_ms": T - t1, "exposed_frac_of_update": (T - t1) / T, "comm_ms": cm,
                   "exposed_frac_of_comm": (T - t1) / cm if cm > 0 else None, "bus_gbs_in_situ": bus,
                   "bus_frac_of_900": bus / 900.0 if bus else None, "ar_launches_per_update": launches,
                   "init_s": init_s}
            st.close()
            if rank == 0:
                print(json.dumps(row), flush=True)
                out.append(row)
        del grads, theta0
        torch.cuda.empty_cache()
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
