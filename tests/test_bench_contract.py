"""bench.py's JSON-line contract, checked on CPU through the reference arm (the unmodified
reference in baseline/_ref when installed, else the oracle port -- test infrastructure, allowed
here): one line with the driver's keys, the reference marker and the cpu_baseline / e2e
objects, and a ms_per_step that the run's own wall clock can contain."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_line(workload, steps=1, warmup=1):
    t0 = time.perf_counter()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          workload, "--steps", str(steps), "--warmup", str(warmup), "--cpu-budget", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    wall = time.perf_counter() - t0
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    # the timed region the line claims must fit in the run that printed it
    assert d["ms_per_step"] * d["steps"] / 1e3 <= wall, (d["ms_per_step"], wall)
    return d


def test_reference_arm_resnet_per_op_sampling():
    d = _ref_line("resnet18-cifar-3pc")
    assert d["impl"] == "reference" and d["value"] > 0
    cb = d["cpu_baseline"]
    if cb["kind"] == "reference":                 # baseline/_ref installed (tools/install_reference.sh)
        assert cb["per_op"] and abs(sum(r["s"] for r in cb["per_op"]) - 1.0 / d["value"]) < 0.01 / d["value"]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "lenet28-3pc", "--steps", "1", "--warmup", "1", "--cpu-budget", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "lenet28-3pc"
