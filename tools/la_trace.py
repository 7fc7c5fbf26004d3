"""Timeline of pipelined host steps (diagnostic): C2 at N=1, four
ts_table_train_steps_host steps with phase timing on; prints every phase
interval (ms from the first event) per stream."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2301_02959_b200 as ts
    args = bench.parse_args([])
    _, ddir, doc = bench.prepare(args, None, 1)
    exp, plan = doc["export"], doc["plan"]
    B = exp["local_batch"]
    batches = []
    for it in range(exp["iterations"]):
        rows = np.fromfile(ddir / f"batch_{it}.rows.u32", np.uint32)
        batches.append(torch.from_numpy(rows.view(np.int32)).pin_memory().numpy().view(np.uint32))
    t = ts.Table(n_rows=exp["n_rows"], dim=exp["embedding_dim"], dp_cut=plan["dp_cut"], flex_cut=plan["flex_cut"],
                 weight_seed=1234, optimizer=ts.OPT_ROWWISE_ADAGRAD, lr=0.01,
                 max_occurrences=max(b.size for b in batches))
    t.train_steps_host(batches)
    t.synchronize()
    t.enable_timing(True)
    t.train_steps_host(batches)
    for name, sid, a, b in t.phase_trace():
        print(f"{name:16s} s{sid} {a:8.3f} {b:8.3f}")
    t.enable_timing(False)
    t.close()


if __name__ == "__main__":
    main()
