"""Multi-GPU parity through NCCL (skipped unless >= 2 GPUs are visible): spawns tests/mp_parity_worker.py."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


def _run(world, family, updates=8, port=29531, impl="auto", graph=False, sharded=False, many=False,
         external=False, acc32=False, split=False):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "tests/mp_parity_worker.py", family,
           str(updates), impl] + (["graph"] if graph else []) + ([sharded if isinstance(sharded, str) else "sharded"] if sharded else []) + \
          (["many"] if many else []) + (["external"] if external else []) + (["acc32"] if acc32 else []) + \
          (["split"] if split else [])
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(p.stdout[-4000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("impl", ["nccl", "fused"])
@pytest.mark.parametrize("family", ["exact", "real"])
def test_world2(family, impl):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, family, port=29531 + (family == "real") + 2 * (impl == "fused"), impl=impl)


@pytest.mark.parametrize("world,graph,ce", [(2, False, 1), (2, True, 1), (4, False, 1), (4, True, 1), (2, True, 2),
                                            (4, False, 2)])
def test_copy_engine_allreduce(world, graph, ce):
    """smpu_config.ar_copy_engine over real NVLink peers: pushes and all-gathers by cudaMemcpyAsync into the other
    ranks' NCCL windows, LSA barriers, the ascending-rank fold; decisions and R bitwise the oracle's (G_real, every
    injection kind), call by call and as one CUDA graph per update."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, "real", port=29581 + 2 * world + graph + 8 * (ce - 1), impl="ce" if ce == 1 else "ce2", graph=graph)


@pytest.mark.parametrize("world", [2, 4])
def test_random_cases_on_real_peers(world):
    """The W > 1 fuzz on real peers (tests/mp_fuzz_worker.py): random layouts, SM / copy-engine / CE-but-last
    all-reduce, pieces, replicated / sharded, injections; decisions and R bitwise the oracle's, replicas identical."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29701 + world), "tests/mp_fuzz_worker.py",
           os.environ.get("SMPU_FUZZ_EXAMPLES", "16" if world == 2 else "10"),
           os.environ.get("SMPU_FUZZ_SEED", str(31 + world))]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=3000)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("impl", ["nccl", "fused"])
def test_world2_cuda_graph(impl):
    """A whole W = 2 update (accumulates, bucket all-reduces, decision exchange, per-bucket Adam) as one graph."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "real", port=29535 + (impl == "fused"), impl=impl, graph=True)


def test_world2_external_accumulation():
    """In-place producer accumulation (smpu_accumulator + micro_grads=None) at W = 2: scans + all-reduces."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "real", port=29538, impl="fused", external=True)


def test_world2_accumulate_many_final_microbatch():
    """smpu_accumulate_many covering the final micro-batch at W = 2 (per-bucket passes + all-reduces)."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "real", port=29539, impl="fused", many=True)


def test_world2_split_tensor_buckets():
    """split_tensors at W = 2: buckets cut through tensors, fused all-reduce per bucket; bitwise the oracle."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "real", port=29571, impl="fused", split=True)


def test_world2_accum_fp32():
    """SURVEY Z1 knob at W = 2: per-rank fp32 sums, rn16, the fused fp16 all-reduce; R bitwise the oracle's
    binary32 variant, decisions bitwise, replicas identical."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "real", port=29567, impl="fused", acc32=True)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_optimizer_bitwise_equals_replicated(world):
    """reduce-scatter + Adam on 1/W + all-gather of w16 agrees bit for bit with the paper's replicated
    update on every rank's shard (theta/m/v) and everywhere (w16), through skips, late decisions and regrowth."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, "real", port=29545 + world, impl="fused", sharded=True)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_optimizer_cuda_graph(world):
    """The launch bench.py times at W > 1: the sharded ctx as one captured CUDA graph per update (device-side
    decision parity, token counts through the pinned ring) agrees bitwise with the replicated call path."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, "real", port=29555 + world, impl="fused", sharded="sharded_graph")


@pytest.mark.parametrize("impl", ["nccl", "fused"])
def test_world4_exact(impl):
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "exact", port=29541 + (impl == "fused"), impl=impl)


def test_world4_real_nccl_decisions():
    """NCCL's fp16 order at W = 4 is not the oracle's (parity unpinned, reading R3): decisions only."""
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "real", port=29543, impl="nccl")


def test_world4_real_fused_bitwise():
    """The fused all-reduce sums in ascending rank order: bitwise the oracle's for G_real at W = 4."""
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "real", port=29544, impl="fused")


def test_c3_enfr_5200_updates_world4():
    """BASELINE configs[3] at the largest W gpurun grants (4): periodic overflow, skip and regrowth."""
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4", "--master-addr",
           "127.0.0.1", "--master-port", "29551", "tests/mp_c3_worker.py", "5200"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("world", [2, 4])
def test_world_invariance_bitwise(world):
    """(W, c=1) through the fused all-reduce == (1, c=W) locally, bit for bit, with G_real (SURVEY c.3)."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29560 + world), "tests/mp_world_invariance_worker.py"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("impl", ["fused", "nccl"])
def test_allreduce_accumulator_primitive(impl):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    world = 4 if _ngpu() >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29570 + (impl == "nccl")), "tests/mp_allreduce_worker.py",
           impl]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


def test_foreign_device_buffer_rejected():
    """A micro-gradient on another GPU than the ctx's is EINVAL, before any state changes (include/smpu.h)."""
    import numpy as np
    import torch
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_1806_00187_b200 as P
    import synth
    from synth import models
    from tests.gpu_util import lib_cfg
    wl = models.Workload("foreign", [("w", 10_000, 0)], 1, 2)
    lay = synth.Layout(wl)
    step = P.UpdateStep(wl.numel, synth.theta0_cpu(wl, lay), lib_cfg(wl), device=0)
    g1 = torch.zeros(lay.n, dtype=torch.int16, device="cuda:1")
    with pytest.raises(P.SmpuError) as ei:
        step.accumulate(g1, 10)
    assert ei.value.status == P.smpu.EINVAL
    g0 = torch.zeros(lay.n, dtype=torch.int16, device="cuda:0")
    step.accumulate(g0, 10)                   # the ctx is unchanged: still two micro-batches to go
    step.accumulate(g0, 10)
    assert step.step()["applied"] == 1
    assert np.isfinite(step.get_master()).all()
    step.close()


def test_mismatched_config_is_einval_on_every_rank():
    """smpu_init compares the collective-shaping config across ranks: a mismatch is EINVAL everywhere, no hang."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29581", "tests/mp_mismatch_worker.py"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
