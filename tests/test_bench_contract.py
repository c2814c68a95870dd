"""bench.py's reference arm on CPU: the JSON line the driver parses (metric,
value, unit, impl, cpu_baseline, e2e, config ...), produced by the unmodified
reference package from baseline/_ref on the C1 fixture (CPU only)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_reference_arm_prints_the_contract_line():
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "ivhd")):
        pytest.skip("reference package not installed in baseline/_ref")
    env = dict(os.environ, RANK="0")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c1",
                        "--steps", "1", "--warmup", "0", "--ref-iters", "2"],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("c1")


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_b200_arm_prints_the_contract_line():
    """The GPU arm on the C1 fixture: roofline, e2e with its copy bytes, gpu
    launches, clocks and the gather floor are present and consistent."""
    env = dict(os.environ, RANK="0")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c1", "--steps", "2",
                        "--warmup", "3", "--no-knn", "--no-cpu", "--no-quality"],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    iters = 2000  # C1: 2000 iterations per step
    assert abs(d["ms_per_step"] * 1e-3 * d["value"] - 3 * 20000 * iters) / (3 * 20000 * iters) < 1e-6
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and 0 < ro["frac"] < 1 and ro["achieved"] > 0 and ro["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 2 * (iters + 1)  # + the deferred decision of each run's last iteration
    assert "sm_mhz" in d["clocks"]  # None when the timed region is shorter than the sampling interval
    assert d["gather_floor"]["us_per_pass"] > 0
