"""GPU planner preview (ts_frontier_preview) against
the authoritative host planner (bit-exact with the reference) on the plan
specs of the parity suite plus a what-if sweep of cost models / topologies:
landmarks and cuts equal, or at most one row apart where the frontier
crosses zero within rounding (the GPU prefix scan sums in another order);
predicted reductions within 1e-9."""
from __future__ import annotations

import pytest

from specs import PLAN_SPECS, TS_DRIVER, run_driver, topo, PAPER_BW

pytestmark = pytest.mark.gpu

SWEEP = [dict(cost_model=dict(local_batch=b, embedding_dim=d)) for b in (256, 1024, 4096) for d in (64, 128)] + \
        [dict(topology=topo(2, 4, PAPER_BW)), dict(topology=topo(4, 8, PAPER_BW)), dict(topology=topo(1, 8)),
         dict(cost_model=dict(local_batch=2048, embedding_dim=128, dp_replication_multiplier=2.0,
                              include_id_bytes=True))]


def check(doc):
    exact = 0
    for entry in doc["preview"]:
        g, h = entry["gpu"], entry["host"]
        for k in ("a", "b", "c", "dp_cut_2tier", "dp_cut_3tier", "flex_cut_3tier"):
            assert abs(g[k] - h[k]) <= 1, (k, g, h)
            exact += g[k] == h[k]
        assert g["c"] == h["c"]  # a threshold count: no summation involved
        # reductions: equal where the cut is equal
        if g["dp_cut_2tier"] == h["dp_cut_2tier"]:
            assert g["reduction_2tier"] == pytest.approx(h["reduction_2tier"], rel=1e-9, abs=1e-12), (g, h)
        if (g["dp_cut_3tier"], g["flex_cut_3tier"]) == (h["dp_cut_3tier"], h["flex_cut_3tier"]):
            assert g["reduction_3tier"] == pytest.approx(h["reduction_3tier"], rel=1e-9, abs=1e-12), (g, h)
    return exact


@pytest.mark.parametrize("name", ["c1_2tier", "c2shape_2x4_3tier", "skew08_2x2_3tier", "skew12_1x4", "skew0_uniform",
                                  "paper_cfg_ids", "no_dyn_mem"])
def test_preview_matches_host_planner(cuda, tmp_path, name):
    spec = dict(PLAN_SPECS[name], frontier=False, preview=dict(what_if=SWEEP))
    doc = run_driver(TS_DRIVER, spec, tmp_path, name)
    assert "error" not in doc, doc
    assert len(doc["preview"]) == 1 + len(SWEEP)
    exact = check(doc)
    assert exact >= 0.9 * 6 * len(doc["preview"])  # nearly all landmarks / cuts identical
