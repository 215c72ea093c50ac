"""The measurement tools regenerate their committed summaries from committed records (CPU only)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c4_summary_from_committed_sweeps(tmp_path):
    out = tmp_path / "c4.txt"
    files = [os.path.join(ROOT, "profiles", "r2", d, f) for d, f in
             (("f_w4", "c4_w4.jsonl"), ("dd_w4", "c4_w2.jsonl"))]
    subprocess.run([sys.executable, "tools/c4_summary.py", str(out)] + files, cwd=ROOT, check=True,
                   capture_output=True)
    txt = out.read_text()
    assert "## W = 4, update_freq = 16" in txt and "## W = 2, update_freq = 1" in txt
    # every C4 threshold of SURVEY 8(d.1) is in the W = 4 sweep
    w4 = txt.split("## W = 4, update_freq = 16")[1].split("##")[0]
    assert [int(l.split()[0]) for l in w4.strip().splitlines()[1:]] == [1, 2, 4, 8, 16, 32, 64, 128, 150, 256]


def test_overlap_model_reproduces_committed_table(tmp_path):
    if not os.path.exists(os.path.join(ROOT, "paper_1806_00187_b200", "libsmpu_sched.so")):
        subprocess.run([sys.executable, os.path.join("paper_1806_00187_b200", "_build.py")], cwd=ROOT, check=True)
    out = tmp_path / "overlap.txt"
    subprocess.run([sys.executable, "tools/overlap_predict.py", str(out)], cwd=ROOT, check=True, capture_output=True)
    assert out.read_text() == open(os.path.join(ROOT, "profiles", "r2_overlap_model.txt")).read()


def test_trace_tail_on_a_synthetic_timeline(tmp_path):
    """tools/trace_tail.py: the last update starts at its k1_first; times relative to the end of its last K1."""
    import json
    ev = [("k1_first", "caller", 0.0, 0.1), ("k1_add", "caller", 0.1, 0.3), ("k2_adam", "adam_per_bucket", 0.3, 0.9),
          ("k1_first", "caller", 1.0, 1.1), ("k1_add", "caller", 1.1, 1.3), ("allreduce", "allreduce", 1.2, 1.6),
          ("k2_adam", "adam_per_bucket", 1.6, 2.0)]
    p = tmp_path / "t.jsonl"
    p.write_text("".join(json.dumps({"rank": 0, "kernel": k, "stream": s, "start_ms": a, "end_ms": b}) + "\n"
                         for k, s, a, b in ev))
    out = subprocess.run([sys.executable, "tools/trace_tail.py", str(p)], cwd=ROOT, check=True, capture_output=True,
                         text=True).stdout
    assert "update 1.000 ms, tail after the last K1 0.700 ms" in out
    assert "'allreduce': 0.3" in out and "'adam_per_bucket': 0.4" in out
