"""The bench.py JSON contract (CPU): the committed bench lines carry every key the driver and the
tier's measurement rules require, and bench.py's argument parser / metric names are consistent."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles", "r1")


def load(name):
    with open(os.path.join(PROF, name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["bench_block1.67M_fp32.json", "bench_block1.67M_fp64.json"])
def test_ours_line_has_the_contract_keys(name):
    d = load(name)
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["metric"] == base["metric"] and d["higher_is_better"] is False and d["warmup"] >= 3
    assert d["config"]["workload"] == "block1.67M"
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    if "cpu_baseline" in d:
        cb = d["cpu_baseline"]
        assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] > 0


def test_reference_line():
    d = load("bench_reference_arm.json")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_cli_parses():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0 and "--impl" in out.stdout and "--gpus" in out.stdout


def test_gpus_flag_spawns_ranks_and_checks_world():
    """`bench.py --gpus N` without a launcher runs N ranks under torch.distributed.run (rank 0 prints);
    under a launcher, WORLD_SIZE != --gpus is an error (the line must not misreport n_gpus)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_arg"] == 2
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=120, env={**env, "WORLD_SIZE": "3"})
    assert bad.returncode == 2 and "WORLD_SIZE" in bad.stderr
