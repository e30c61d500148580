"""bench.py keeps the driver's JSON-line contract (keys, types, units)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def run_bench(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [line for line in out.stdout.splitlines() if line.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_json_contract():
    d = run_bench("--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "2", "--settle", "0")
    for k, typ in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                   ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                   ("dtype", str), ("data", str), ("config", dict), ("e2e", dict), ("roofline", dict),
                   ("gpu_launches", int), ("clocks", dict)):
        assert isinstance(d[k], typ), k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["vs_baseline"] is None
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] == 2 * 5
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.05 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)


def test_bench_configs_run():
    for cfg in ("1", "4"):
        d = run_bench("--config", cfg, "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                      "--settle", "0")
        assert d["value"] > 0 and d["e2e"] is None
