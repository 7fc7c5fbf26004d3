"""simulate() parity: the product (ts_driver: host planner + GPU routing
kernel, csrc/device/router.cu) against the compiled reference
(oracle/_ref/ref_driver) — every SimReport field of every iteration, the RW
baseline, compare_to_baseline and compare(), bit-exact (== on doubles).
Also the router C-ABI alone against the restated counters of the committed
golden fixture (tests/golden/mini_2x4_3tier.npz)."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_bind as orc
from specs import REF_DRIVER, SIM_SPECS, TS_DRIVER, run_driver, strip

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", sorted(SIM_SPECS))
def test_simulate_matches_reference(cuda, name, tmp_path):
    spec = SIM_SPECS[name]
    mine = strip(run_driver(TS_DRIVER, spec, tmp_path, name))
    assert "error" not in mine, mine
    golden = GOLDEN / f"{name}.ref.json"
    if REF_DRIVER.exists():
        ref = strip(run_driver(REF_DRIVER, spec, tmp_path, name))
    else:
        ref = json.loads(golden.read_text())
    assert mine.keys() == ref.keys()
    for key in ref:
        assert mine[key] == ref[key], f"{name}: field {key} differs"


def test_router_counters_match_golden(cuda):
    import paper_2301_02959_b200 as ts
    g = np.load(GOLDEN / "mini_2x4_3tier.npz")
    n_nodes, w = int(g["num_nodes"]), int(g["gpus_per_node"])
    dest = np.where(g["tier"] == 1, g["slot"], g["owner"]).astype(np.uint8)
    router = ts.Router(len(dest), int(g["dp_cut"]), int(g["flex_cut"]), dest, n_nodes, w)
    for it in range(int(g["iterations"])):
        got = router.iteration(int(g["local_batch"]), g[f"offsets_{it}"], g[f"rows_{it}"])
        assert np.array_equal(got, g[f"counters_{it}"]), f"iteration {it}"
    # a row outside the plan is rejected, not silently routed
    bad = g["rows_0"].copy()
    bad[0] = len(dest)
    with pytest.raises(ts.TSError) as e:
        router.iteration(int(g["local_batch"]), g["offsets_0"], bad)
    assert e.value.kind == "ValidationError"
    router.close()
