"""Host planner parity: the product's C++ API (ts_driver over
libtiershard_b200.so) against the compiled reference — distribution order
digest, breakpoints, frontier landmarks and samples, cuts, CostReport,
coverage, placement digest.  Doubles compared with == (bit-exact)."""
import json
from pathlib import Path

import pytest

from specs import PLAN_SPECS, REF_DRIVER, TS_DRIVER, run_driver, strip

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", sorted(PLAN_SPECS))
def test_plan_matches_reference(name, tmp_path):
    spec = PLAN_SPECS[name]
    mine = strip(run_driver(TS_DRIVER, spec, tmp_path, name))
    ref = json.loads((GOLDEN / f"{name}.ref.json").read_text())
    assert "error" not in mine, mine
    assert mine.keys() == ref.keys()
    for key in ref:
        assert mine[key] == ref[key], f"{name}: {key}"


def test_hash_and_rng_match_reference(tmp_path):
    mine = run_driver(TS_DRIVER, {"hash_vectors": True}, tmp_path, "hash")["hash"]
    ref = json.loads((GOLDEN / "hash_vectors.json").read_text())
    assert mine == ref


@pytest.mark.parametrize("spec,kind", [
    (dict(tables=[dict(rows=10, exponent=1.0, target_length=1, seed=1)],
          topology=dict(num_nodes=1, gpus_per_node=2, a2a_global_gibs=2, a2a_intra_gibs=1,
                        ar_global_gibs=1, ar_cross_gibs=1)), "ConfigError"),
    (dict(tables=[dict(rows=0, exponent=1.0, target_length=1, seed=1)],
          topology=dict(num_nodes=1, gpus_per_node=1, a2a_global_gibs=1, a2a_intra_gibs=1,
                        ar_global_gibs=1, ar_cross_gibs=1)), "ConfigError"),
    (dict(tables=[dict(rows=100, exponent=1.0, target_length=1, seed=1)],
          topology=dict(num_nodes=1, gpus_per_node=1, a2a_global_gibs=1, a2a_intra_gibs=1,
                        ar_global_gibs=1, ar_cross_gibs=1), goal="budget", budget_bytes=-1e30), "ValidationError"),
    (dict(tables=[dict(table_id=0, rows=100, exponent=1.0, target_length=1, seed=1),
                  dict(table_id=0, rows=100, exponent=1.0, target_length=1, seed=2)],
          topology=dict(num_nodes=1, gpus_per_node=1, a2a_global_gibs=1, a2a_intra_gibs=1,
                        ar_global_gibs=1, ar_cross_gibs=1)), "ValidationError"),
])
def test_errors_match_reference(spec, kind, tmp_path):
    mine = run_driver(TS_DRIVER, spec, tmp_path, "err")
    assert mine.get("error") == kind
    if REF_DRIVER.exists():
        ref = run_driver(REF_DRIVER, spec, tmp_path, "err")
        assert ref == {k: v for k, v in mine.items()}, (ref, mine)
