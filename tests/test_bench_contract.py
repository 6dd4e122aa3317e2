"""bench.py's reference arm on CPU: one JSON line with the driver's keys, the
b200 arm's workload / metric / unit, and its own cpu_baseline and e2e
objects (the reference's own step when baseline/_ref holds it, else the oracle
port; run here on a 1-step sample of config 5, one member per host core)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--spinup", "0"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600, check=True).stdout
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["unit"] == "cell-steps/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "config5" and d["config"]["mode"] == "adaptive"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "nhswe")):
        assert cb["kind"] == "reference"
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_cpu_leg_falls_back_to_the_oracle_port(monkeypatch):
    """Without baseline/_ref the CPU legs run the oracle port (labelled
    "port"); with it, the reference's own adaptive_step ("reference")."""
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setenv("NH_CPU_ARM", "port")
    cells, secs, kind = bench._cpu_worker(("config4", 1, 1, 2, "adaptive"))
    assert kind == "port" and cells == 2 * 4096 and secs > 0
    monkeypatch.delenv("NH_CPU_ARM")
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "nhswe")):
        assert bench._cpu_worker(("config4", 1, 1, 2, "adaptive"))[2] == "reference"
