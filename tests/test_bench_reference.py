"""bench.py's reference arm (the CPU oracle, this tier's `--impl reference`) honours the driver's JSON contract:
one line with impl, metric, value, unit, the timing keys, cpu_baseline and a zero-copy e2e; runs without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "2",
                        "--warmup", "1", "--ref-seconds", "1.5"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "grad elems/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "tiny" and d["config"]["n_params"] == 1_000_000


def test_reference_arm_under_torchrun_prints_once():
    """Launched as the driver launches N > 1 (torchrun, 2 ranks, no GPU needed): rank 0 alone prints the line."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29613", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--config", "tiny", "--steps", "2", "--warmup", "1", "--ref-seconds", "1.5"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["world"] == 2


def test_self_launch_without_torchrun_prints_once():
    """`bench.py --gpus 2` with no WORLD_SIZE spawns its own two ranks (127.0.0.1 rendezvous): one line, exit 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "tiny",
                        "--steps", "2", "--warmup", "1", "--ref-seconds", "1.5"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["world"] == 2


def test_reference_arm_timing_fits_the_run_and_mirrors_config():
    """ms_per_step is measured (not extrapolated): steps x ms_per_step fits inside the run's wall time; the config
    carries the repo arm's keys."""
    import time
    t0 = time.perf_counter()
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "3",
                        "--warmup", "1", "--ref-seconds", "2"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    wall = time.perf_counter() - t0
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["steps"] * d["ms_per_step"] / 1000 < wall
    for key in ("workload", "n_params", "n_tensors", "update_freq", "world", "bucket_mib", "n_buckets",
                "tokens_per_update", "generator", "parallelism", "fuse_final", "accum_fp32", "path_bytes_per_elem",
                "optimizer", "l2"):
        assert key in d["config"], key
    assert d["config"]["n_buckets"] == 1 and d["config"]["optimizer"] == "replicated (paper)"
