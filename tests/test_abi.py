"""The C ABI library loads and exports every symbol include/smpu.h declares; host-only calls (no GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from synth import models

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    so = os.path.join(ROOT, "paper_1806_00187_b200", "libsmpu.so")
    if not os.path.exists(so):
        import subprocess
        import sys
        subprocess.run([sys.executable, os.path.join("paper_1806_00187_b200", "_build.py")], cwd=ROOT, check=True)
    import paper_1806_00187_b200 as pkg
    return pkg


def header_functions():
    src = open(os.path.join(ROOT, "include", "smpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(smpu_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(P):
    names = header_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(P.smpu.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(P.smpu.EXPORTS)   # the binding covers the whole header


def test_abi_version_and_defaults(P):
    assert P.abi_version() == 4
    c = P.config_default()
    # fuse_final is opt-in: the default ctx keeps SURVEY 8(b)'s contract (w16 changes only inside smpu_step)
    assert (c.allreduce, c.sharded, c.fuse_final, c.accum_fp32, c.split_tensors) == (0, 0, 0, 0, 0)
    assert (c.peak_lr, c.warmup_updates, c.beta1, c.beta2, c.eps) == (5e-4, 4000, 0.9, 0.98, 1e-8)
    assert (c.init_scale_log2, c.min_scale_log2, c.max_scale_log2, c.growth_interval) == (7, -5, 24, 2000)
    assert c.bucket_bytes == 150 << 20                                                                # P:212 fn
    # the fused all-reduce's shape lives in the config (compared across ranks at init), not in the environment
    assert (c.ar_ctas, c.ar_threads, c.ar_vec_bytes, c.ar_unroll, c.ar_mcast, c.pdl) == (0, 256, 32, 1, 0, 1)
    assert (c.ar_pieces, c.ar_copy_engine) == (1, 0)


def test_library_reads_no_environment_knobs():
    """Collective shape knobs come from smpu_config only (a rank with a different environment would otherwise pick
    a different LSA barrier count or multicast requirement and hang its peers)."""
    src = open(os.path.join(ROOT, "paper_1806_00187_b200", "csrc", "smpu.cu")).read()
    assert not re.findall(r'getenv\("SMPU_(AR_|PDL)', src)


# whole-tensor greedy buckets of Transformer-big En-De (count, last bucket MiB)
A2 = {1: (61, 64.0), 2: (61, 64.0), 4: (43, 64.0), 8: (43, 64.0), 16: (22, 64.0), 32: (11, 80.0), 64: (6, 80.0),
      128: (3, 144.1), 150: (3, 96.0), 256: (2, 144.1)}


@pytest.mark.parametrize("mib", sorted(A2))
def test_bucket_plan_big_ende(P, mib):
    wl = models.big_ende()
    b = P.plan_buckets(wl.numel, mib << 20)
    nb, last = A2[mib]
    assert len(b) - 1 == nb
    assert round((b[-1] - b[-2]) * 2 / 2**20, 1) == last
    assert b[0] == 0 and b[-1] == wl.n
    # every bucket but the last reaches the threshold; boundaries are tensor boundaries (whole tensors)
    sizes = np.diff(b) * 2
    assert np.all(sizes[:-1] >= mib << 20)
    ends = set(np.cumsum(wl.numel).tolist())
    assert all(int(x) in ends for x in b[1:])


def test_bucket_plan_150mib_paper_configs(P):
    # "150MB" buckets: big En-De 152.2/152.2/96.0 MiB, big En-Fr 152.2/152.2/119.0, base 1 x 116.2
    mib = lambda b: [round(x * 2 / 2**20, 1) for x in np.diff(b)]  # noqa: E731
    assert mib(P.plan_buckets(models.big_ende().numel, 150 << 20)) == [152.2, 152.2, 96.0]
    assert mib(P.plan_buckets(models.big_enfr().numel, 150 << 20)) == [152.2, 152.2, 119.0]
    assert mib(P.plan_buckets(models.base_ende().numel, 150 << 20)) == [116.2]


def test_bucket_plan_rejects_bad_input(P):
    with pytest.raises(P.SmpuError) as ei:
        P.plan_buckets([10, 0, 5], 100)
    assert ei.value.status == P.smpu.EINVAL


def test_product_has_no_oracle_dependency():
    # the product path never imports / links the oracle (task rule)
    pkg = os.path.join(ROOT, "paper_1806_00187_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle-exact", ""), f


def test_sched_library_exports_header():
    so = os.path.join(ROOT, "paper_1806_00187_b200", "libsmpu_sched.so")
    if not os.path.exists(so):
        import subprocess
        import sys
        subprocess.run([sys.executable, os.path.join("paper_1806_00187_b200", "_build.py")], cwd=ROOT, check=True)
    src = open(os.path.join(ROOT, "include", "smpu_sched.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(smpu_sched_[a-z_]+)\s*\(", src)))
    assert len(names) == 6   # token_budget, fit_timing, estimate, time_balanced, simulate, overlap_schedule
    lib = ctypes.CDLL(so)
    for name in names:
        assert hasattr(lib, name), name


def test_kernel_ids_match_header(P):
    """The binding's kernel-id table is the header's enum (smpu_kernel_stats indexes by it)."""
    hdr = open(os.path.join(ROOT, "include", "smpu.h")).read()
    ids = {m.group(1): int(m.group(2)) for m in re.finditer(r"SMPU_(K\w+|ALLREDUCE|DECISION_AR|N_KERNELS) = (\d+)", hdr)}
    assert ids["N_KERNELS"] == P.smpu.N_KERNELS == len(P.smpu.KERNEL_NAMES)
    for name, k in ids.items():
        if name != "N_KERNELS":
            assert getattr(P.smpu, name) == k, name


def test_struct_layouts_match_header(P, tmp_path):
    """The ctypes mirrors of smpu_config / smpu_step_result have the C layout: offsets and sizes printed by a C
    program compiled against include/smpu.h (a field added on one side only would shift every later field)."""
    import subprocess
    src = tmp_path / "layout.c"
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "smpu.h"', "int main(void) {"]
    for cname, py in (("smpu_config", P.smpu.Config), ("smpu_step_result", P.smpu.StepResult)):
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], check=True, capture_output=True,
                                                        text=True).stdout.splitlines())
    for cname, py in (("smpu_config", P.smpu.Config), ("smpu_step_result", P.smpu.StepResult)):
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"


def test_missing_library_is_an_import_error(tmp_path):
    """No silent fallback: the package without its built libsmpu.so refuses to import."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_1806_00187_b200"
    pkg.mkdir()
    for f in os.listdir(os.path.join(ROOT, "paper_1806_00187_b200")):
        if f.endswith(".py"):
            shutil.copy(os.path.join(ROOT, "paper_1806_00187_b200", f), pkg / f)
    r = subprocess.run([sys.executable, "-c", "import paper_1806_00187_b200"], cwd=tmp_path, capture_output=True,
                       text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr and "no CPU fallback" in r.stderr


@pytest.mark.parametrize("world", [2, 3, 4, 5, 6, 7, 8])
def test_shard_plan_partitions_every_bucket(P, world):
    """Host logic of the sharded layout at every world size the peer kernels take, W = 8 included
    (gpurun grants at most 4 GPUs): the ranks' ranges cover every element exactly once, stay inside their
    bucket, are 8-element aligned except rank 0's bucket heads / tails, and split each bucket's units evenly."""
    rng = np.random.default_rng(world)
    for trial in range(20):
        numel = rng.integers(1, 5000, rng.integers(1, 12))
        bb = P.plan_buckets(numel, int(rng.choice([2, 100, 3000, 20000])))
        n = int(bb[-1])
        mark = np.zeros(n, np.int32)
        for r in range(world):
            for lo, hi in P.smpu.plan_shards(bb, world, r):
                assert 0 <= lo < hi <= n
                b = int(np.searchsorted(bb, lo, side="right")) - 1
                assert hi <= bb[b + 1], "a range crosses a bucket boundary"
                if r > 0:
                    assert lo % 8 == 0 and hi % 8 == 0
                mark[lo:hi] += 1
        assert (mark == 1).all(), (trial, world)
        for b in range(len(bb) - 1):                        # the aligned units are split evenly
            v0, v1 = (bb[b] + 7) // 8 * 8, bb[b + 1] // 8 * 8
            units = max(v1 - v0, 0) // 8
            per = -(-units // world)
            sizes = [sum(min(h, v1) - max(l, v0) for l, h in P.smpu.plan_shards(bb[b:b + 2], world, r)
                         if min(h, v1) > max(l, v0)) // 8 for r in range(world)]
            assert sum(sizes) == units and max(sizes, default=0) <= per


def test_config_and_group_argument_errors_need_no_gpu(P):
    """Argument checks run before any CUDA call: a bad all-reduce shape, and virtual groups outside 2..8 ranks, with
    the NCCL all-reduce, or with NVLS multicast, are EINVAL (include/smpu.h)."""
    wl = models.Workload("args", [("w", 1000, 0)], 1, 1)
    theta0 = np.zeros(1000, np.float32)
    for bad in (dict(ar_threads=300), dict(ar_vec_bytes=8), dict(ar_unroll=3), dict(ar_ctas=-1), dict(pdl=2),
                dict(ar_mcast=1, ar_vec_bytes=16), dict(ar_copy_engine=3), dict(ar_copy_engine=1, sharded=1),
                dict(ar_copy_engine=1, ar_mcast=1), dict(ar_copy_engine=1, allreduce=P.smpu.AR_NCCL)):
        with pytest.raises(P.SmpuError) as ei:
            P.UpdateStep(wl.numel, theta0, P.config_default(**bad))
        assert ei.value.status == P.smpu.EINVAL, bad
    for world, kw in ((1, {}), (9, {}), (2, dict(allreduce=P.smpu.AR_NCCL)), (2, dict(ar_mcast=1))):
        with pytest.raises(P.SmpuError) as ei:
            P.VirtualGroup(wl.numel, theta0, P.config_default(**kw), world=world)
        assert ei.value.status == P.smpu.EINVAL, (world, kw)
