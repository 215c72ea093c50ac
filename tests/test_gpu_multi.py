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


def _run(world, family, updates=8, port=29531):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "tests/mp_parity_worker.py", family,
           str(updates)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(p.stdout[-4000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


@pytest.mark.parametrize("family", ["exact", "real"])
def test_world2(family):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, family, port=29531 if family == "exact" else 29532)


def test_world4_exact():
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "exact", port=29533)


def test_world4_real_decisions():
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, "real", port=29534)
