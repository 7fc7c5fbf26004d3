"""C3 skew sweep (BASELINE.json configs[2]): for Zipf
exponents {0, 0.8, 1.05, 1.2} at 2 / 4 / 8 GPUs (1 x U homogeneous, 2-tier)
and 2 x 4 virtual nodes (paper bandwidths, 3-tier), the all-to-all bytes the
FlexShard plan moves against row-wise (hash) and table-wise sharding of the
same tables on the same sampled iteration.  C2 table shapes (8 x 10M rows,
D = 128, L = 128 per table, batch 4096 per GPU).  Host only: the planner and
placement are the product's (bit-exact with the reference); traffic is
counted per occurrence by bin/ts_driver's export.

    python tools/skew_sweep.py OUT.json [--rows N]
"""
import argparse
import json
import subprocess
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
DRIVER = ROOT / "paper_2301_02959_b200" / "bin" / "ts_driver"
HOMO = dict(a2a_global_gibs=1, a2a_intra_gibs=1, ar_global_gibs=1, ar_cross_gibs=1)
PAPER_BW = dict(a2a_global_gibs=23, a2a_intra_gibs=95, ar_global_gibs=73, ar_cross_gibs=15)


def run(alpha, nodes, w, goal, bw, rows, tmp):
    spec = dict(tables=[dict(table_id=t, rows=rows, exponent=alpha, target_length=128, seed=1000 + t)
                        for t in range(8)],
                topology=dict(num_nodes=nodes, gpus_per_node=w, **bw),
                cost_model=dict(local_batch=4096, embedding_dim=128), goal=goal, frontier=False,
                hash_seed=2, workload=dict(seed=7, iterations=1), export_dir=str(tmp))
    (tmp / "spec.json").write_text(json.dumps(spec))
    subprocess.run([str(DRIVER), str(tmp / "spec.json"), str(tmp / "doc.json")], check=True)
    doc = json.loads((tmp / "doc.json").read_text())
    tr = doc["export"]["traffic"][0]
    ref, off = tr["reference_convention"], tr["off_device"]
    plan_off = off["plan_global_bytes"] + off["plan_intra_bytes"]
    return {
        "exponent": alpha, "topology": f"{nodes}x{w}", "goal": goal, "gpus": nodes * w,
        "dp_cut": doc["plan"]["dp_cut"], "flex_cut": doc["plan"]["flex_cut"],
        "predicted_global_a2a_reduction": doc["plan"]["predicted"]["global_a2a_reduction"],
        "measured_global_a2a_reduction": 1 - ref["plan_global_bytes"] / ref["rw_global_bytes"],
        "occurrences": tr["occurrences"],
        "off_device_GB": {"plan": plan_off / 1e9, "rw": off["rw_bytes"] / 1e9, "tw": off["tw_bytes"] / 1e9},
        "saved_vs_rw_GB": (off["rw_bytes"] - plan_off) / 1e9,
        "saved_vs_tw_GB": (off["tw_bytes"] - plan_off) / 1e9,
        "max_send_GB": {k: v / 1e9 for k, v in tr["max_send_bytes"].items()},
        "max_send_off_device_GB": {k: v / 1e9 for k, v in tr["max_send_off_device_bytes"].items()},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--rows", type=int, default=10_000_000)
    args = ap.parse_args()
    res = []
    with tempfile.TemporaryDirectory() as td:
        for alpha in (0.0, 0.8, 1.05, 1.2):
            for nodes, w, goal, bw in ((1, 2, "2tier", HOMO), (1, 4, "2tier", HOMO), (1, 8, "2tier", HOMO),
                                       (2, 4, "3tier", PAPER_BW)):
                r = run(alpha, nodes, w, goal, bw, args.rows, Path(td))
                res.append(r)
                print(f"alpha={alpha:4} {r['topology']} {goal}: dp={r['dp_cut']} flex={r['flex_cut'] - r['dp_cut']} "
                      f"reduction pred={r['predicted_global_a2a_reduction']:.4f} "
                      f"meas={r['measured_global_a2a_reduction']:.4f} off-device GB plan/rw/tw = "
                      f"{r['off_device_GB']['plan']:.3f}/{r['off_device_GB']['rw']:.3f}/{r['off_device_GB']['tw']:.3f} "
                      f"max-send off-device GB plan/rw/tw = " + "/".join(f"{r['max_send_off_device_GB'][k]:.3f}" for k in ("plan", "rw", "tw")),
                      flush=True)
    Path(args.out).write_text(json.dumps(dict(
        description=__doc__.strip().splitlines()[0], rows_per_table=args.rows, results=res), indent=1) + "\n")


if __name__ == "__main__":
    main()
