"""Routing-kernel probe (diagnostic): one logical C2 iteration at U = 8
(1 x 8 or 2 x 4) routed K times through ts_router_iteration_device; prints
the median kernel time.  Used for A/B runs and ncu captures:

    python tools/route_probe.py [--topo 1x8|2x4] [--iters K]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--topo", default="1x8")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2301_02959_b200 as ts
    args = bench.parse_args([])
    args.iterations, args.virtual_nodes = 1, a.topo == "2x4"
    _, ddir, doc = bench.prepare(args, None, 8)
    exp, plan = doc["export"], doc["plan"]
    u, w, B = exp["num_gpus"], exp["gpus_per_node"], exp["local_batch"]
    dest = np.fromfile(ddir / "dest.u8", np.uint8)
    rows = np.fromfile(ddir / "batch_0.rows.u32", np.uint32)
    off = np.fromfile(ddir / "batch_0.offsets.u64", np.uint64)
    bounds = np.ascontiguousarray(off[np.arange(u + 1) * B])
    router = ts.Router(exp["n_rows"], plan["dp_cut"], plan["flex_cut"], dest, u // w, w)
    d_rows = torch.from_numpy(rows.view(np.int32)).cuda()
    d_b = torch.from_numpy(bounds.view(np.int64)).cuda()
    ks = []
    for _ in range(a.iters):
        c = router.iteration_device(d_b.data_ptr(), d_rows.data_ptr(), rows.size)
        ks.append(router.last_timing()[0])
    print(f"{a.topo}: occ={rows.size} kernel_ms median={np.median(ks):.4f} min={min(ks):.4f} "
          f"counters_sum={int(c.sum())}")


if __name__ == "__main__":
    main()
