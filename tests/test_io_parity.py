"""Manifest / plan-document / CSV parity (json_io.hpp, manifest.hpp).

One client source (paper_2301_02959_b200/csrc/tools/artifacts_main.cpp) is
compiled against our library (bin/ts_artifacts) and against the unmodified
reference (oracle/_ref/ref_artifacts).  Both read the same manifest and write
plan.json, frontier/coverage/assignment CSVs and (with sim_iterations > 0)
the simulation artefacts; every file must be byte-identical.  Where the
reference build is absent the files are checked against the sha256 digests in
tests/golden/io_digests.json, generated from the reference by
tests/golden/make_golden.py --io.

The simulation artefacts need the GPU router (our simulate() has no CPU
fallback), so the CPU cases set sim_iterations = 0 and the `gpu` case runs
the full manifest.
"""
from __future__ import annotations

import hashlib
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
TS_ARTIFACTS = ROOT / "paper_2301_02959_b200" / "bin" / "ts_artifacts"
REF_ARTIFACTS = ROOT / "oracle" / "_ref" / "ref_artifacts"
DIGESTS = Path(__file__).resolve().parent / "golden" / "io_digests.json"

TOPO_2X4 = dict(num_nodes=2, gpus_per_node=4, a2a_global_gibs=12.5, a2a_intra_gibs=150,
                ar_global_gibs=20, ar_cross_gibs=25)
TOPO_1X8 = dict(num_nodes=1, gpus_per_node=8, a2a_global_gibs=100, a2a_intra_gibs=100,
                ar_global_gibs=80, ar_cross_gibs=80)


def histogram_text(rows: int, step: int, seed: int) -> str:
    """Deterministic sparse histogram (row_id,count) with fractional counts."""
    lines = ["row_id,count"]
    x = seed
    for r in range(0, rows, step):
        x = (x * 6364136223846793005 + 1442695040888963407) % (1 << 64)
        lines.append(f"{r},{(x >> 40) % 41 + ((x >> 20) % 4) * 0.25}")
    return "\n".join(lines) + "\n"


# name -> (manifest, topology, {histogram file: text})
CASES = {
    "mixed_3tier": (
        dict(topology="topo.json", cost_model=dict(local_batch=64, embedding_dim=32),
             tables=[dict(table_id=0, rows=3000, zipf=dict(exponent=1.1, target_length=20)),
                     dict(table_id=5, rows=600, histogram="h5.csv", num_samples=1000)],
             plan="3tier", seed=11, sim_iterations=3),
        TOPO_2X4, {"h5.csv": histogram_text(600, 3, 5)}),
    "zipf_2tier_1x8": (
        dict(topology="topo.json", cost_model=dict(local_batch=512, embedding_dim=64),
             tables=[dict(table_id=t, rows=20000, zipf=dict(exponent=1.05, target_length=32))
                     for t in range(3)],
             plan="2tier", seed=2, sim_iterations=2),
        TOPO_1X8, {}),
    "budget_flex": (
        dict(topology="topo.json", cost_model=dict(local_batch=256, embedding_dim=64),
             tables=[dict(table_id=1, rows=10000, zipf=dict(exponent=1.2, target_length=40))],
             plan="budget:2e6", budget_allow_flex=True, seed=5, hash_seed=99, sim_iterations=2),
        TOPO_2X4, {}),
    "frontier_hist": (
        dict(topology="topo.json",
             cost_model=dict(local_batch=128, embedding_dim=16, include_id_bytes=True),
             tables=[dict(table_id=2, rows=900, histogram="h2.csv", num_samples=4096),
                     dict(table_id=3, rows=700, histogram="h3.csv", num_samples=2048)],
             plan="frontier", seed=9, sim_iterations=2),
        TOPO_2X4, {"h2.csv": histogram_text(900, 2, 2), "h3.csv": histogram_text(700, 5, 3)}),
}

# name -> (manifest, topology or None, files)
ERROR_CASES = {
    "missing_topology": (dict(tables=[]), None, {}),
    "duplicate_table": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, zipf=dict(exponent=1, target_length=1)),
                                           dict(table_id=1, rows=10, zipf=dict(exponent=1, target_length=1))]),
        TOPO_2X4, {}),
    "zipf_and_histogram": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, histogram="h.csv", num_samples=4,
                                                zipf=dict(exponent=1, target_length=1))]),
        TOPO_2X4, {"h.csv": "row_id,count\n1,2\n"}),
    "histogram_no_samples": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, histogram="h.csv")]),
        TOPO_2X4, {"h.csv": "row_id,count\n1,2\n"}),
    "no_tables": (dict(topology="topo.json"), TOPO_2X4, {}),
    "table_without_rows": (dict(topology="topo.json", tables=[dict(table_id=1)]), TOPO_2X4, {}),
    "degenerate_topology": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, zipf=dict(exponent=1, target_length=1))]),
        dict(TOPO_2X4, a2a_intra_gibs=1), {}),
    "topology_missing_field": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, zipf=dict(exponent=1, target_length=1))]),
        {k: v for k, v in TOPO_2X4.items() if k != "ar_cross_gibs"}, {}),
    "histogram_row_out_of_range": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, histogram="h.csv", num_samples=8)]),
        TOPO_2X4, {"h.csv": "row_id,count\n3,1\n12,1\n"}),
    "histogram_bad_header": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, histogram="h.csv", num_samples=8)]),
        TOPO_2X4, {"h.csv": "id,count\n3,1\n"}),
    "histogram_missing_file": (
        dict(topology="topo.json", tables=[dict(table_id=1, rows=10, histogram="nope.csv", num_samples=8)]),
        TOPO_2X4, {}),
    "bad_cost_model": (
        dict(topology="topo.json", cost_model=dict(embedding_dim=0),
             tables=[dict(table_id=1, rows=10, zipf=dict(exponent=1, target_length=1))]),
        TOPO_2X4, {}),
    "unknown_goal": (
        dict(topology="topo.json", plan="4tier",
             tables=[dict(table_id=1, rows=10, zipf=dict(exponent=1, target_length=1))]),
        TOPO_2X4, {}),
}


def write_case(base: Path, manifest: dict, topo: dict | None, files: dict, sim: bool) -> Path:
    base.mkdir(parents=True, exist_ok=True)
    m = dict(manifest)
    if not sim and "sim_iterations" in m:
        m["sim_iterations"] = 0
    (base / "manifest.json").write_text(json.dumps(m))
    if topo is not None:
        (base / "topo.json").write_text(json.dumps(topo))
    for name, text in files.items():
        (base / name).write_text(text)
    return base / "manifest.json"


def run_artifacts(exe: Path, manifest: Path, out: Path) -> tuple[int, dict[str, bytes]]:
    proc = subprocess.run([str(exe), str(manifest), str(out), "4"], capture_output=True, timeout=600)
    files = {p.name: p.read_bytes() for p in sorted(out.iterdir())} if out.exists() else {}
    return proc.returncode, files


def digests(files: dict[str, bytes]) -> dict[str, str]:
    return {k: hashlib.sha256(v).hexdigest() for k, v in files.items()}


def check_against_reference(key: str, code: int, files: dict[str, bytes], tmp_path: Path,
                            manifest: Path):
    if REF_ARTIFACTS.exists():
        ref_code, ref_files = run_artifacts(REF_ARTIFACTS, manifest, tmp_path / "ref")
        assert code == ref_code, (files.get("error.txt"), ref_files.get("error.txt"))
        assert sorted(files) == sorted(ref_files)
        for name in ref_files:
            assert files[name] == ref_files[name], f"{key}: {name} differs from the reference"
    golden = json.loads(DIGESTS.read_text())
    assert key in golden, f"no golden digests for {key}; run tests/golden/make_golden.py --io"
    assert digests(files) == golden[key]


@pytest.mark.parametrize("name", sorted(CASES))
def test_artifacts_byte_identical(name, tmp_path):
    manifest = write_case(tmp_path / "in", *CASES[name], sim=False)
    code, files = run_artifacts(TS_ARTIFACTS, manifest, tmp_path / "ours")
    assert code == 0, files.get("error.txt")
    assert {"plan.json", "plan_reloaded.json", "frontier.csv", "coverage.csv", "coverage.txt",
            "assignment.csv"} <= set(files)
    # load_plan_document + save_plan_document is a fixed point.
    assert files["plan.json"] == files["plan_reloaded.json"]
    check_against_reference(f"{name}/nosim", code, files, tmp_path, manifest)


@pytest.mark.parametrize("name", sorted(ERROR_CASES))
def test_manifest_errors_match_reference(name, tmp_path):
    manifest = write_case(tmp_path / "in", *ERROR_CASES[name], sim=False)
    code, files = run_artifacts(TS_ARTIFACTS, manifest, tmp_path / "ours")
    assert code == 3 and "error.txt" in files, files.keys()
    # Paths inside messages are tmp-dir specific: compare live, and the
    # golden form with the directory replaced.
    if REF_ARTIFACTS.exists():
        ref_code, ref_files = run_artifacts(REF_ARTIFACTS, manifest, tmp_path / "ref")
        assert ref_code == code
        assert ref_files == files
    golden = json.loads(DIGESTS.read_text())
    text = files["error.txt"].decode().replace(str(tmp_path / "in"), "<dir>")
    assert golden[f"error/{name}"] == text


def test_plan_document_loader_rejects_bad_documents(tmp_path):
    """load_plan_document: invalid JSON and degenerate topologies are
    ConfigErrors (json_io.cpp:276-318 in the reference)."""
    manifest = write_case(tmp_path / "in", *CASES["zipf_2tier_1x8"], sim=False)
    code, files = run_artifacts(TS_ARTIFACTS, manifest, tmp_path / "ours")
    assert code == 0
    doc = json.loads(files["plan.json"])
    assert doc["tool_version"] == "0.1.0"
    assert doc["dp_cut"] == len(doc["dp_rows"])
    assert doc["flex_cut"] - doc["dp_cut"] == len(doc["flex_rows"])
    assert set(doc["points"]) == {"a", "b", "c", "d"}
    rows = files["assignment.csv"].decode().splitlines()
    assert rows[0] == "table_id,row_id,tier"
    assert len(rows) - 1 == doc["total_rows"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_sim_artifacts_byte_identical(name, tmp_path, cuda):
    manifest = write_case(tmp_path / "in", *CASES[name], sim=True)
    code, files = run_artifacts(TS_ARTIFACTS, manifest, tmp_path / "ours")
    assert code == 0, files.get("error.txt")
    assert {"sim.csv", "sim_report.json", "discrepancies.json"} <= set(files)
    check_against_reference(f"{name}/sim", code, files, tmp_path, manifest)
