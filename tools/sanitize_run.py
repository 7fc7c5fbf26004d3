"""Small workloads for compute-sanitizer (diagnostic): the U = 1 train step
(gather, dedup sort, short / long segment paths, Adagrad) and the U = 2 peer
step on ONE GPU through the in-process group (route, request pull, serve,
gradient push, replicated-row reduction), plus the router.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch
    import paper_2301_02959_b200 as ts
    import mg_worker

    # U = 1: Zipf batch with hot rows (multi-piece segments) and a cold tail
    n, dim, occ = 50_000, 128, 40_000
    rng = np.random.default_rng(3)
    p = np.arange(1, n + 1, dtype=np.float64) ** -1.1
    rows = rng.choice(n, size=occ, p=p / p.sum()).astype(np.uint32)
    t = ts.Table(n_rows=n, dim=dim, dp_cut=500, flex_cut=500, optimizer=ts.OPT_ROWWISE_ADAGRAD, lr=0.01,
                 max_occurrences=occ)
    d_rows = torch.from_numpy(rows.view(np.int32)).cuda()
    d_out = torch.empty((occ, dim), dtype=torch.float32, device="cuda")
    for _ in range(2):
        t.train_step(d_rows.data_ptr(), occ, d_out.data_ptr())
    t.train_step_host(rows[: occ // 2])
    t.synchronize()
    t.counters()
    t.read_rows(np.arange(0, n, 7, dtype=np.uint32), with_state=True)
    t.close()
    print("u1 ok", flush=True)

    # U = 2 (and 2 x 2) peer path on one device, several steps
    for nodes, w in ((1, 2), (2, 2)):
        mg_worker.run_inproc(nodes, w, 1, 1e-4, steps=3, pipelined=True)
        mg_worker.run_inproc(nodes, w, 0, 1e-3, steps=1)
        print(f"inproc {nodes}x{w} ok", flush=True)

    # router, logical 2 x 4
    u, wpn = 8, 4
    tier, owner, slot = __import__("oracle_bind").assign_rows(np.zeros(n, np.uint32), np.arange(n, dtype=np.uint64),
                                                              300, 3000, u, wpn, 2)
    dest = np.where(tier == 1, slot, owner).astype(np.uint8)
    r = ts.Router(n, 300, 3000, dest, 2, wpn)
    batch = rng.choice(n, size=8 * 4000, p=p / p.sum()).astype(np.uint32)
    offs = np.arange(0, 8 * 4000 + 1, 4000, dtype=np.uint64)
    r.iteration(1, offs, batch)
    r.close()
    print("router ok", flush=True)


if __name__ == "__main__":
    main()
