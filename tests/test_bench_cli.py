"""bench.py contract checks that need no GPU: the reference arm prints one JSON
line with the driver's keys (it times the reference compiled in oracle/_ref)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbcs_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "0", "--size", "20"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # measured on the named system itself (no extrapolation): steps = calls timed
    assert d["steps"] == len(d["step_times_s"]) >= 1 and "20^3" in d["config"]["workload"]
    assert d["cpu_baseline"]["host"]["nproc"] >= 1


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbcs_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_under_torchrun_ranks():
    """Under torchrun (N > 1) only rank 0 runs the reference and prints; the
    other ranks exit 0 without output (the driver launches both arms alike)."""
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
            "--size", "12", "--gpus", "2"]
    env = dict(os.environ, WORLD_SIZE="2", LOCAL_RANK="1", RANK="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29555")
    out = subprocess.run(base, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    assert not [l for l in out.stdout.splitlines() if l.strip()]
    env.update(LOCAL_RANK="0", RANK="0")
    out = subprocess.run(base, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and "per-GPU share" in d["cpu_baseline"]["sample"]
