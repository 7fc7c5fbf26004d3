"""Generates the committed golden fixtures under tests/golden/ by running the
UNMODIFIED reference (oracle/_ref/ref_driver, compiled from /root/reference by
oracle/Makefile).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Outputs
  <name>.ref.json      reference document for every spec in tests/specs.py
                       (SIM_SPECS and PLAN_SPECS), timing stripped
  hash_vectors.json    mix64 / row_key_hash / derive_seed / SplitMix64 /
                       Poisson known answers
  mini_2x4_3tier.npz   placements, 4 iterations of batches and the per-GPU
                       counter block of each iteration (restated counters,
                       verified here against the reference's SimReport)
  c2_full_*.ref.json   (--c2) full-C2 simulate() documents (tests/specs.py
                       C2_SIM_SPECS)
  io_digests.json      (--io) sha256 of every artefact oracle/_ref/ref_artifacts
                       writes for tests/test_io_parity.py's manifests, and
                       the reference's error text for each malformed one
"""
from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_bind as orc  # noqa: E402
from specs import C2_SIM_SPECS, PLAN_SPECS, REF_DRIVER, SIM_SPECS, run_driver, strip  # noqa: E402


def make_c2() -> None:
    """Full-C2 simulate() documents (long: ~1-2 min of reference time each)."""
    with tempfile.TemporaryDirectory() as td:
        for name, spec in C2_SIM_SPECS.items():
            doc = strip(run_driver(REF_DRIVER, spec, Path(td), name))
            (HERE / f"{name}.ref.json").write_text(json.dumps(doc) + "\n")
            print("wrote", name)


def main() -> None:
    assert REF_DRIVER.exists(), "build oracle/_ref first: make -C oracle ref"
    with tempfile.TemporaryDirectory() as td:
        tmp = Path(td)
        doc = run_driver(REF_DRIVER, {"hash_vectors": True}, tmp, "hash")
        (HERE / "hash_vectors.json").write_text(json.dumps(doc["hash"], indent=1) + "\n")
        for name, spec in {**PLAN_SPECS, **SIM_SPECS}.items():
            doc = strip(run_driver(REF_DRIVER, spec, tmp, name))
            (HERE / f"{name}.ref.json").write_text(json.dumps(doc) + "\n")
            print("wrote", name)

        # binary fixture for the router C-ABI test
        name = "mini_2x4_3tier"
        spec = dict(SIM_SPECS[name])
        dump = tmp / "dump"
        dump.mkdir()
        spec["dump_dir"] = str(dump)
        spec["workload"] = dict(spec["workload"], dump_batches=True)
        doc = run_driver(REF_DRIVER, spec, tmp, name + "_dump")
        topo = spec["topology"]
        n_nodes, w = topo["num_nodes"], topo["gpus_per_node"]
        u = n_nodes * w
        tier = np.fromfile(dump / "placements.tier.u8", np.uint8)
        owner = np.fromfile(dump / "placements.owner.u32", np.uint32)
        slot = np.fromfile(dump / "placements.slot.u32", np.uint32)
        b = spec["cost_model"]["local_batch"]
        out = dict(num_nodes=n_nodes, gpus_per_node=w, local_batch=b,
                   dp_cut=doc["plan"]["dp_cut"], flex_cut=doc["plan"]["flex_cut"],
                   iterations=spec["workload"]["iterations"], tier=tier, owner=owner, slot=slot)
        row_bytes = spec["cost_model"]["embedding_dim"] * 4
        for it in range(spec["workload"]["iterations"]):
            rows = np.fromfile(dump / f"batch_{it}.rows.u32", np.uint32)
            off = np.fromfile(dump / f"batch_{it}.offsets.u64", np.uint64)
            cnt = orc.route_counts(u, w, b, off, rows, tier, owner, slot)
            # pin the restatement: its metrics must equal the reference's
            flex_rows = slot[doc["plan"]["dp_cut"]:doc["plan"]["flex_cut"]]
            per_slot = np.bincount(flex_rows, minlength=w) if flex_rows.size else np.zeros(w, int)
            gib = 1073741824.0
            m = orc.iteration_metrics(
                cnt, dim=spec["cost_model"]["embedding_dim"], include_id=False,
                bw=(topo["a2a_global_gibs"] * gib, topo["a2a_intra_gibs"] * gib,
                    topo["ar_global_gibs"] * gib, topo["ar_cross_gibs"] * gib),
                ar_global_bytes=float(doc["plan"]["dp_cut"]) * row_bytes,
                ar_cross_max=float(per_slot.max()) * row_bytes,
                ar_cross_mean=float(per_slot.sum()) / w * row_bytes)
            ref_m = doc["sim"]["iterations"][it]
            assert m == ref_m, (it, {k: (m[k], ref_m[k]) for k in m if m[k] != ref_m[k]})
            out[f"rows_{it}"] = rows
            out[f"offsets_{it}"] = off
            out[f"counters_{it}"] = cnt
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print("wrote", name + ".npz")


def make_io_digests() -> None:
    import test_io_parity as io
    assert io.REF_ARTIFACTS.exists(), "build oracle/_ref first: make -C oracle ref"
    golden = {}
    with tempfile.TemporaryDirectory() as td:
        tmp = Path(td)
        for name, case in io.CASES.items():
            for sim in (False, True):
                base = tmp / name / ("sim" if sim else "nosim")
                manifest = io.write_case(base / "in", *case, sim=sim)
                code, files = io.run_artifacts(io.REF_ARTIFACTS, manifest, base / "out")
                assert code == 0, files.get("error.txt")
                golden[f"{name}/{'sim' if sim else 'nosim'}"] = io.digests(files)
        for name, case in io.ERROR_CASES.items():
            base = tmp / "err" / name
            manifest = io.write_case(base / "in", *case, sim=False)
            code, files = io.run_artifacts(io.REF_ARTIFACTS, manifest, base / "out")
            assert code == 3, (name, code)
            golden[f"error/{name}"] = files["error.txt"].decode().replace(str(base / "in"), "<dir>")
    (HERE / "io_digests.json").write_text(json.dumps(golden, indent=1, sort_keys=True) + "\n")
    print("wrote io_digests.json")


if __name__ == "__main__":
    if "--io" in sys.argv:
        make_io_digests()
    elif "--c2" in sys.argv:
        make_c2()
    else:
        main()
