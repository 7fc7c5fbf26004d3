"""Multi-GPU probe in ONE process (diagnostic): U ranks as threads over a
ts_group, rank g on GPU g, the C2 workload at 1 x U (bench.py's prepared
batches), K device-resident train steps.  One process, so ncu can capture
the exchange kernels' NVLink counters (nvlrx / nvltx bytes) per launch:

    python tools/mg_probe.py --gpus 2 --steps 3
"""
import argparse
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--virtual-nodes", action="store_true")
    a = ap.parse_args()
    import torch
    import bench
    import paper_2301_02959_b200 as ts

    args = bench.parse_args([])
    args.iterations, args.virtual_nodes = 1, a.virtual_nodes
    _, ddir, doc = bench.prepare(args, None, a.gpus)
    exp, plan = doc["export"], doc["plan"]
    u, w, B, D = exp["num_gpus"], exp["gpus_per_node"], exp["local_batch"], exp["embedding_dim"]
    dest = np.fromfile(ddir / "dest.u8", np.uint8)
    rows = np.fromfile(ddir / "batch_0.rows.u32", np.uint32)
    off = np.fromfile(ddir / "batch_0.offsets.u64", np.uint64)
    most = max(t["max_send_off_device_bytes"]["plan"] for t in exp["traffic"]) / (D * 4)
    grp = ts.Group(u)
    ms = [None] * u
    errors = []

    def rank(g):
        try:
            torch.cuda.set_device(g)
            lo, hi = int(off[g * B]), int(off[(g + 1) * B])
            b = np.ascontiguousarray(rows[lo:hi])
            t = ts.Table(n_rows=exp["n_rows"], dim=D, dp_cut=plan["dp_cut"], flex_cut=plan["flex_cut"],
                         tier_dest=dest, num_nodes=u // w, gpus_per_node=w, rank=g, device=g, weight_seed=1234,
                         optimizer=ts.OPT_ROWWISE_ADAGRAD, lr=0.01, max_occurrences=b.size,
                         recv_rows_hint=int(most * 1.25) + 4096, group=grp)
            d_rows = torch.from_numpy(b.view(np.int32)).cuda()
            d_out = torch.empty((b.size, D), dtype=torch.float32, device="cuda")
            t.train_step(d_rows.data_ptr(), b.size, d_out.data_ptr())
            t.synchronize()
            t0 = time.perf_counter()
            for _ in range(a.steps):
                t.train_step(d_rows.data_ptr(), b.size, d_out.data_ptr())
            t.synchronize()
            ms[g] = (time.perf_counter() - t0) * 1e3 / a.steps
            t.close()
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            grp.abort()

    th = [threading.Thread(target=rank, args=(g,)) for g in range(u)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    if errors:
        raise errors[0]
    grp.close()
    print(f"in-process {u // w}x{w}: wall ms/step per rank {['%.3f' % m for m in ms]} (host-timed, incl. launch)")


if __name__ == "__main__":
    main()
