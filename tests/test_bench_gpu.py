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
    d = run_bench("--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "2", "--settle", "0",
                  "--sustain-s", "0.2")
    for k, typ in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                   ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                   ("dtype", str), ("data", str), ("config", dict), ("e2e", dict), ("roofline", dict),
                   ("gpu_launches", int), ("clocks", dict)):
        assert isinstance(d[k], typ), k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["vs_baseline"] is None
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] == 2 * 5  # K1, K2 (20x25 pads: the fp64 kernel)
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.05 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["parity"]["ok"] and d["parity"]["rgb_max_lsb"] <= 1 and d["parity"]["mask_mismatches"] == 0
    assert len(d["validation"]["sha256"]) == 64 and d["validation"]["frames"] == 8192
    assert d["value_sustained"] > 0 and d["sustained"]["seconds"] >= 0.15
    oc = d["other_configs"]  # configs 4 and 5, briefly, with their parity blocks
    assert set(oc) == {"4", "5"}
    for k, o in oc.items():
        assert o["value"] > 0 and o["parity"]["ok"] and 0 < o["kernel_frac_of_hbm_peak"] < 1.05, k


def test_bench_configs_run():
    for cfg in ("1", "4"):
        d = run_bench("--config", cfg, "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                      "--settle", "0", "--also", "")
        assert d["value"] > 0 and d["e2e"] is None


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_match_one_rank():
    """bench.py under torchrun with 2 ranks (gloo for the collectives, both
    ranks on the one GPU of this box -- a functional check of the sharding and
    of the validation gather, not a measurement): the gathered parity block is
    green and the whole-job digest equals the N=1 run's."""
    import os
    common = ["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--settle", "0",
              "--sustain-s", "0", "--envs", "512", "--also", ""]
    one = run_bench(*common)
    env = dict(os.environ, TACSL_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                          str(ROOT / "bench.py"), "--gpus", "2", *common],
                         capture_output=True, text=True, cwd=ROOT, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [line for line in out.stdout.splitlines() if line.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    two = json.loads(lines[0])
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert one["parity"]["ok"] and two["parity"]["ok"], (one["parity"], two["parity"])
    assert two["validation"]["sha256"] == one["validation"]["sha256"]
    assert two["validation"]["frames"] == one["validation"]["frames"] == 1024
    for k in ("rgb_max_lsb", "rgb_frac_off", "ff_max_rel", "mask_mismatches", "frames_checked"):
        assert two["parity"][k] == one["parity"][k], k
