"""The `tiershard` command-line front end (bin/tiershard; SURVEY.md §8(f)
row 3, SPEC.md `cli` module): plan artefacts byte-identical to the
reference's json_io output for the same manifest, deterministic reruns,
histogram synth round trip, error exits; `simulate` on the GPU."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

import test_io_parity as io

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2301_02959_b200" / "bin" / "tiershard"


def cli(*args, cwd=None):
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=600, cwd=cwd)


def ref_files(tmp_path: Path, name: str, sim: bool) -> dict[str, bytes]:
    manifest = io.write_case(tmp_path / "refin", *io.CASES[name], sim=sim)
    exe = io.REF_ARTIFACTS if io.REF_ARTIFACTS.exists() else io.TS_ARTIFACTS
    code, files = io.run_artifacts(exe, manifest, tmp_path / "ref")
    assert code == 0, files.get("error.txt")
    return files


@pytest.mark.parametrize("name", sorted(io.CASES))
def test_plan_artifacts_match_reference(name, tmp_path):
    manifest = io.write_case(tmp_path / "in", *io.CASES[name], sim=False)
    p = cli("plan", "--manifest", manifest, "--out", tmp_path / "out")
    assert p.returncode == 0, p.stderr
    ref = ref_files(tmp_path, name, sim=False)
    for f in ("plan.json", "frontier.csv", "coverage.csv", "assignment.csv"):
        assert (tmp_path / "out" / f).read_bytes() == ref[f], f
    assert p.stdout.encode() == ref["coverage.txt"]
    # rerun: byte-identical
    p2 = cli("plan", "--manifest", manifest, "--out", tmp_path / "out2")
    for f in ("plan.json", "frontier.csv", "coverage.csv", "assignment.csv"):
        assert (tmp_path / "out" / f).read_bytes() == (tmp_path / "out2" / f).read_bytes()


def test_default_output_dir_is_relative_to_manifest(tmp_path):
    m, topo, files = io.CASES["zipf_2tier_1x8"]
    manifest = io.write_case(tmp_path / "in", dict(m, output_dir="results"), topo, files, sim=False)
    p = cli("plan", "--manifest", manifest, cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    assert (tmp_path / "in" / "results" / "plan.json").exists()


def test_synth_round_trip(tmp_path):
    """Synthesized histograms reloaded through a histogram manifest give the
    same plan as the Zipf manifest (counts = p * 2^20 round-trip exactly)."""
    m, topo, files = io.CASES["zipf_2tier_1x8"]
    manifest = io.write_case(tmp_path / "in", m, topo, files, sim=False)
    p = cli("synth", "--manifest", manifest, "--out", tmp_path / "in" / "syn")
    assert p.returncode == 0, p.stderr
    echo = json.loads((tmp_path / "in" / "syn" / "manifest_echo.json").read_text())
    hist = dict(m, tables=[dict(table_id=t["table_id"], rows=t["rows"], histogram="syn/" + t["histogram"],
                                num_samples=t["num_samples"]) for t in echo["tables"]])
    (tmp_path / "in" / "hist.json").write_text(json.dumps(dict(hist, sim_iterations=0)))
    a = cli("plan", "--manifest", manifest, "--out", tmp_path / "a")
    b = cli("plan", "--manifest", tmp_path / "in" / "hist.json", "--out", tmp_path / "b")
    assert a.returncode == 0 and b.returncode == 0, b.stderr
    da = json.loads((tmp_path / "a" / "plan.json").read_text())
    db = json.loads((tmp_path / "b" / "plan.json").read_text())
    for k in ("dp_cut", "flex_cut", "total_rows", "dp_rows", "flex_rows", "predicted", "capacity"):
        assert da[k] == db[k], k
    assert (tmp_path / "a" / "assignment.csv").read_bytes() == (tmp_path / "b" / "assignment.csv").read_bytes()
    # same seed: byte-identical synth output
    p2 = cli("synth", "--manifest", manifest, "--out", tmp_path / "syn2")
    for t in echo["tables"]:
        f = t["histogram"]
        assert (tmp_path / "in" / "syn" / f).read_bytes() == (tmp_path / "syn2" / f).read_bytes()


def test_breakpoints(tmp_path):
    manifest = io.write_case(tmp_path / "in", *io.CASES["mixed_3tier"], sim=False)
    p = cli("breakpoints", "--manifest", manifest)
    assert p.returncode == 0, p.stderr
    bp = json.loads(p.stdout)
    assert set(bp) == {"p_mem_dp", "p_comm_dp", "flex_mem_price_bytes", "p_comm_flex"}
    assert bp["p_mem_dp"] > bp["p_comm_dp"] > 0


def test_errors(tmp_path):
    p = cli("plan", "--manifest", tmp_path / "missing.json")
    assert p.returncode == 3 and "manifest: cannot open" in p.stderr
    p = cli("frobnicate", "--manifest", tmp_path / "missing.json")
    assert p.returncode == 2 and "unknown command" in p.stderr
    p = cli("plan")
    assert p.returncode == 2 and "--manifest is required" in p.stderr
    (tmp_path / "topo.json").write_text(json.dumps(io.TOPO_2X4))
    (tmp_path / "empty.json").write_text(json.dumps(dict(topology="topo.json")))
    p = cli("synth", "--manifest", tmp_path / "empty.json")
    assert p.returncode == 3 and "empty manifest" in p.stderr
    manifest = io.write_case(tmp_path / "in", *io.CASES["zipf_2tier_1x8"], sim=False)
    p = cli("simulate", "--manifest", manifest, "--plan", tmp_path / "nope.json", "--out", tmp_path / "o")
    assert p.returncode == 3 and "plan: cannot open" in p.stderr


def test_simulate_rejects_mismatched_plan(tmp_path):
    a = io.write_case(tmp_path / "a", *io.CASES["zipf_2tier_1x8"], sim=False)
    b = io.write_case(tmp_path / "b", *io.CASES["budget_flex"], sim=False)
    assert cli("plan", "--manifest", a, "--out", tmp_path / "pa").returncode == 0
    p = cli("simulate", "--manifest", b, "--plan", tmp_path / "pa" / "plan.json", "--out", tmp_path / "o")
    assert p.returncode == 3 and "does not match the manifest" in p.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mixed_3tier", "budget_flex"])
def test_simulate_matches_reference(name, tmp_path, cuda):
    manifest = io.write_case(tmp_path / "in", *io.CASES[name], sim=True)
    assert cli("plan", "--manifest", manifest, "--out", tmp_path / "out").returncode == 0
    p = cli("simulate", "--manifest", manifest, "--out", tmp_path / "out", "--threads", 4)
    assert p.returncode == 0, p.stderr
    ref = ref_files(tmp_path, name, sim=True)
    for f in ("sim_report.json", "sim.csv", "discrepancies.json"):
        assert (tmp_path / "out" / f).read_bytes() == ref[f], f
    assert "reduction" in p.stdout
    c = cli("compare", "--manifest", manifest, "--out", tmp_path / "out")
    assert c.returncode == 0 and "global_a2a" in c.stdout


def test_preview_fails_loudly_without_device(tmp_path):
    import paper_2301_02959_b200 as ts
    if ts.device_count() > 0:
        pytest.skip("a device is present")
    manifest = io.write_case(tmp_path / "in", *io.CASES["zipf_2tier_1x8"], sim=False)
    p = cli("preview", "--manifest", manifest)
    assert p.returncode == 3 and "no CUDA device" in p.stderr


@pytest.mark.gpu
def test_preview_sweep(tmp_path, cuda):
    manifest = io.write_case(tmp_path / "in", *io.CASES["mixed_3tier"], sim=False)
    assert cli("plan", "--manifest", manifest, "--out", tmp_path / "out").returncode == 0
    doc = json.loads((tmp_path / "out" / "plan.json").read_text())
    sweep = [dict(cost_model=dict(local_batch=b)) for b in (16, 64, 256)] + \
            [dict(topology=dict(num_nodes=4, gpus_per_node=8))]
    (tmp_path / "sweep.json").write_text(json.dumps(sweep))
    p = cli("preview", "--manifest", manifest, "--plan", tmp_path / "sweep.json")
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout)
    assert len(out) == 1 + len(sweep)
    first = out[0]["plan_3tier"]  # the manifest's own 3-tier plan
    assert abs(first["dp_cut"] - doc["dp_cut"]) <= 1 and abs(first["flex_cut"] - doc["flex_cut"]) <= 1
    assert [o["cost_model"]["local_batch"] for o in out[1:4]] == [16, 64, 256]
    # larger batches make more rows worth replicating
    assert out[1]["plan_2tier"]["dp_cut"] <= out[2]["plan_2tier"]["dp_cut"] <= out[3]["plan_2tier"]["dp_cut"]
