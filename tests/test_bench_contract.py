"""bench.py's driver contract, checked on the CPU at a small size:
  * `--impl reference` runs the unmodified reference (oracle/_ref) and prints
    ONE JSON line with the contract's keys (impl, metric, value, unit,
    higher_is_better, cpu_baseline with kind / cores / sample, e2e);
  * our arm has no CPU fallback: without a GPU it exits non-zero with the
    library's NoDevice error instead of printing a number."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SMALL = ["--tables", "2", "--rows", "20000", "--batch", "64", "--seq-len", "16"]


def run_bench(*args, timeout=600):
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_reference_arm_contract(tmp_path):
    if not (ROOT / "oracle" / "_ref" / "ref_driver").exists():
        pytest.skip("reference build absent (needs /root/reference)")
    p = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--cache", str(tmp_path), *SMALL)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "samples/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # like for like: routing + accounting only (the pool's sampling time is
    # subtracted), and the exact config dict our arm prints for this workload
    t = d["reference_timing"]
    assert 0 < t["materialize_parallel_s"] < t["simulate_s"]
    assert d["value_including_sampling"] < d["value"]
    sys.path.insert(0, str(ROOT))
    import bench
    ns = bench.parse_args(SMALL)
    c = d["config"]
    assert c == bench.job_config(ns, 1, 1, c["plan"], c["dp_cut"], c["flex_cut"])


def test_our_arm_has_no_cpu_fallback(tmp_path):
    import paper_2301_02959_b200 as ts
    if ts.device_count() > 0:
        pytest.skip("a device is present")
    p = run_bench("--steps", "1", "--warmup", "1", "--no-cpu-baseline", "--no-e2e", "--cache", str(tmp_path),
                  *SMALL)
    assert p.returncode != 0
    assert not [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert "NoDevice" in p.stderr or "no CUDA device" in p.stderr
