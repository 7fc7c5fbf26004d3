"""Shared spec documents (the ref_driver / ts_driver JSON format,
oracle/README.md) for the parity tests and the golden-fixture generator."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_DRIVER = ROOT / "oracle" / "_ref" / "ref_driver"
TS_DRIVER = ROOT / "paper_2301_02959_b200" / "bin" / "ts_driver"

HOMO = dict(a2a_global_gibs=1, a2a_intra_gibs=1, ar_global_gibs=1, ar_cross_gibs=1)
PAPER_BW = dict(a2a_global_gibs=23, a2a_intra_gibs=95, ar_global_gibs=73, ar_cross_gibs=15)


def topo(n, w, bw=HOMO):
    return dict(num_nodes=n, gpus_per_node=w, **bw)


def tables(count, rows, exponent, length, seed0=1000):
    return [dict(table_id=t, rows=rows, exponent=exponent, target_length=length, seed=seed0 + t)
            for t in range(count)]


# name -> spec.  Sizes keep each reference run to a few seconds.
PLAN_SPECS = {
    "c1_2tier": dict(tables=[dict(table_id=0, rows=1_000_000, exponent=1.05, target_length=32, seed=1)],
                     topology=topo(1, 1), cost_model=dict(local_batch=256, embedding_dim=64), goal="2tier"),
    "c2shape_1x8_2tier": dict(tables=tables(8, 200_000, 1.05, 128), topology=topo(1, 8),
                              cost_model=dict(local_batch=4096, embedding_dim=128), goal="2tier"),
    "c2shape_2x4_3tier": dict(tables=tables(8, 200_000, 1.05, 128), topology=topo(2, 4, PAPER_BW),
                              cost_model=dict(local_batch=4096, embedding_dim=128), goal="3tier"),
    "skew0_uniform": dict(tables=tables(2, 50_000, 0.0, 64), topology=topo(1, 2),
                          cost_model=dict(local_batch=1024, embedding_dim=128), goal="2tier"),
    "skew08_2x2_3tier": dict(tables=tables(4, 50_000, 0.8, 128), topology=topo(2, 2, PAPER_BW),
                             cost_model=dict(local_batch=2048, embedding_dim=128), goal="3tier"),
    "skew12_1x4": dict(tables=tables(4, 50_000, 1.2, 128), topology=topo(1, 4),
                       cost_model=dict(local_batch=2048, embedding_dim=128), goal="2tier"),
    "budget_neg": dict(tables=tables(2, 40_000, 1.05, 100), topology=topo(2, 2, PAPER_BW),
                       cost_model=dict(local_batch=1024, embedding_dim=64), goal="budget",
                       budget_bytes=-2.0e6, allow_flex=False),
    "budget_flex": dict(tables=tables(2, 40_000, 1.05, 100), topology=topo(2, 2, PAPER_BW),
                        cost_model=dict(local_batch=1024, embedding_dim=64), goal="budget",
                        budget_bytes=0.0, allow_flex=True),
    "paper_cfg_ids": dict(tables=tables(4, 30_000, 1.05, 1000), topology=topo(4, 8, PAPER_BW),
                          cost_model=dict(local_batch=64, embedding_dim=256, include_id_bytes=True),
                          goal="3tier"),
    "no_dyn_mem": dict(tables=tables(2, 30_000, 1.05, 50), topology=topo(1, 4),
                       cost_model=dict(local_batch=512, embedding_dim=32, count_dynamic_memory=False),
                       goal="budget", budget_bytes=1.0e5, allow_flex=False),
}

# Simulation specs (routing on the GPU in ts_driver).
SIM_SPECS = {
    "c1_sim": dict(PLAN_SPECS["c1_2tier"], workload=dict(seed=7, iterations=3), baseline=True),
    "mini_2x4_3tier": dict(tables=tables(4, 30_000, 1.05, 64), topology=topo(2, 4, PAPER_BW),
                           cost_model=dict(local_batch=64, embedding_dim=128), goal="3tier",
                           workload=dict(seed=7, iterations=4), baseline=True, threads=4),
    "mini_1x8_2tier": dict(tables=tables(2, 40_000, 1.05, 96), topology=topo(1, 8),
                           cost_model=dict(local_batch=32, embedding_dim=64), goal="2tier",
                           workload=dict(seed=11, iterations=3), baseline=True, threads=2),
    "mini_rw_u4": dict(tables=tables(2, 20_000, 1.2, 64), topology=topo(2, 2),
                       cost_model=dict(local_batch=32, embedding_dim=64), goal="rw",
                       workload=dict(seed=3, iterations=2)),
    "mini_uniform": dict(tables=tables(1, 10_000, 0.0, 40), topology=topo(1, 2),
                         cost_model=dict(local_batch=16, embedding_dim=32), goal="2tier",
                         workload=dict(seed=5, iterations=2)),
    "paper_desk_ids": dict(tables=[dict(table_id=0, rows=30_000, exponent=1.05, target_length=1000, seed=1),
                                   dict(table_id=1, rows=30_000, exponent=1.05, target_length=1000, seed=2),
                                   dict(table_id=2, rows=10_000, exponent=1.05, target_length=500, seed=3),
                                   dict(table_id=3, rows=10_000, exponent=1.05, target_length=500, seed=4)],
                           topology=topo(4, 8, PAPER_BW),
                           cost_model=dict(local_batch=64, embedding_dim=256, include_id_bytes=True),
                           goal="3tier", workload=dict(seed=9, iterations=2), baseline=True, threads=2),
}

# Full C2 (BASELINE configs[1]: 8 tables x 10M rows, D=128, L=128/table,
# B=4096/GPU) at logical U=8, one sampled iteration: the routing loop at the
# scale the bench runs (33.6M occurrences).  ~1-2 min per reference run.
C2_SIM_SPECS = {
    "c2_full_1x8_2tier": dict(tables=tables(8, 10_000_000, 1.05, 128), topology=topo(1, 8),
                              cost_model=dict(local_batch=4096, embedding_dim=128), goal="2tier",
                              workload=dict(seed=7, iterations=1), threads=8),
    "c2_full_2x4_3tier": dict(tables=tables(8, 10_000_000, 1.05, 128), topology=topo(2, 4, PAPER_BW),
                              cost_model=dict(local_batch=4096, embedding_dim=128), goal="3tier",
                              workload=dict(seed=7, iterations=1), threads=8),
}


def run_driver(driver: Path, spec: dict, workdir: Path, name: str) -> dict:
    spec_path = workdir / f"{name}.spec.json"
    spec_path.write_text(json.dumps(spec))
    out_path = workdir / f"{name}.{driver.name}.json"
    proc = subprocess.run([str(driver), str(spec_path), str(out_path)], capture_output=True, text=True,
                          timeout=900)
    if proc.returncode not in (0, 3):
        raise RuntimeError(f"{driver.name} failed rc={proc.returncode}: {proc.stderr[-2000:]}")
    return json.loads(out_path.read_text())


def strip(doc: dict) -> dict:
    return {k: v for k, v in doc.items() if k not in ("tool", "timing")}
