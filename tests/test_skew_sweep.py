"""C3 skew sweep (BASELINE.json configs[2]): the all-to-all
bytes the FlexShard plan moves against row-wise and table-wise sharding.

Two checks, host only:
* tools/skew_sweep.py runs from its tools/ location through bin/ts_driver on
  a scaled-down table, and the counted traffic agrees with the planner's
  prediction (the model-identity property, SPEC acceptance 4);
* the committed full-size sweep (profiles/r02_skew_sweep.json) keeps the same
  properties, so the bytes-saved figures DESIGN.md quotes are self-consistent.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import skew_sweep  # noqa: E402

PROFILE = ROOT / "profiles" / "r02_skew_sweep.json"


def check_row(r: dict) -> None:
    # counted global a2a reduction equals the planner's prediction
    assert abs(r["measured_global_a2a_reduction"] - r["predicted_global_a2a_reduction"]) < 5e-4, r
    off = r["off_device_GB"]
    # the plan never moves more than row-wise sharding; with no hot tier it
    # is row-wise (table-wise can then come out a few sampled rows lower)
    assert off["plan"] <= off["rw"] + 1e-9, r
    if r["flex_cut"] == 0:
        assert off["plan"] == pytest.approx(off["rw"], abs=1e-9)
    else:
        assert off["plan"] < off["tw"], r
    assert r["saved_vs_rw_GB"] == pytest.approx(off["rw"] - off["plan"], abs=1e-9)
    assert r["saved_vs_tw_GB"] == pytest.approx(off["tw"] - off["plan"], abs=1e-9)
    assert r["dp_cut"] <= r["flex_cut"]
    # the critical path: the most loaded server's off-device sends.  The plan
    # never loads a server more than row-wise does, and with a hot tier it is
    # below table-wise as well (hot rows are served on every GPU)
    ms = r.get("max_send_off_device_GB")
    if ms is not None:
        assert ms["plan"] <= ms["rw"] + 1e-9, r
        if r["flex_cut"] > 0:
            assert ms["plan"] < ms["tw"], r
    if r["goal"] == "2tier":
        assert r["dp_cut"] == r["flex_cut"]


@pytest.mark.parametrize("nodes,w,goal,bw", [(1, 4, "2tier", skew_sweep.HOMO),
                                             (2, 2, "3tier", skew_sweep.PAPER_BW)])
def test_sweep_point_runs(nodes, w, goal, bw, tmp_path):
    if not skew_sweep.DRIVER.exists():
        pytest.fail(f"{skew_sweep.DRIVER} missing: run __graft_entry__.build()")
    r = skew_sweep.run(1.05, nodes, w, goal, bw, 200_000, tmp_path)
    check_row(r)
    assert r["gpus"] == nodes * w and r["topology"] == f"{nodes}x{w}"
    # a skewed table gets a non-trivial hot tier and saves most of the traffic
    assert r["flex_cut"] > 0 and r["measured_global_a2a_reduction"] > 0.5
    if goal == "3tier":
        assert r["dp_cut"] < r["flex_cut"]


def test_committed_sweep_consistent():
    doc = json.loads(PROFILE.read_text())
    assert doc["rows_per_table"] == 10_000_000
    rows = doc["results"]
    assert {r["exponent"] for r in rows} == {0.0, 0.8, 1.05, 1.2}
    assert {r["topology"] for r in rows} == {"1x2", "1x4", "1x8", "2x4"}
    for r in rows:
        check_row(r)
    # uniform rows get no hot tier; more skew never saves less (per topology)
    for topo in ("1x2", "1x4", "1x8", "2x4"):
        series = sorted((r for r in rows if r["topology"] == topo), key=lambda r: r["exponent"])
        assert series[0]["flex_cut"] == 0
        red = [r["measured_global_a2a_reduction"] for r in series]
        assert red[1] < red[2], (topo, red)
