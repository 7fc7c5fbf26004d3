"""Rank worker for tests/test_gpu_multigpu.py (launched by torch.distributed.run,
one process per GPU).  Runs one forward + backward of a U-rank sharded table
through the C-ABI over NCCL and dumps what it saw for the parent test to
check against the oracle."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def problem(n_nodes, w, seed=11, steps=1):
    """rows[g] is rank g's first batch; steps > 1 adds steps_rows[s][g] for
    the host-API multi-step case, batches growing step to step (so any
    per-step buffer sized by the batch would have to move)."""
    import oracle_bind as orc
    u = n_nodes * w
    n, dim = 12000, 64
    dp_cut, flex_cut = 150, 1500 if n_nodes * w > 1 else 150
    rng = np.random.default_rng(seed)
    p = np.arange(1, n + 1, dtype=np.float64) ** -1.1
    occ = [int(x) for x in rng.integers(3000, 6000, size=u)]
    rows = [rng.choice(n, size=o, p=p / p.sum()).astype(np.uint32) for o in occ]
    steps_rows = [rows]
    for s in range(1, steps):
        steps_rows.append([rng.choice(n, size=o + 1500 * s, p=p / p.sum()).astype(np.uint32) for o in occ])
    tier, owner, slot = orc.assign_rows(np.zeros(n, np.uint32), np.arange(n, dtype=np.uint64),
                                        dp_cut, flex_cut, u, w, 2)
    dest = np.where(tier == 1, slot, owner).astype(np.uint8)
    return dict(n=n, dim=dim, dp_cut=dp_cut, flex_cut=flex_cut, rows=rows, tier=tier, owner=owner,
                slot=slot, dest=dest, steps_rows=steps_rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, required=True)
    ap.add_argument("--gpus-per-node", type=int, required=True)
    ap.add_argument("--optimizer", type=int, default=1)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--steps", type=int, default=1, help="> 1: host-buffer steps (train_step_host)")
    ap.add_argument("--pipelined", action="store_true", help="the steps in one train_steps_host call")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import torch
    import torch.distributed as td
    import paper_2301_02959_b200 as ts

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo")
    assert world == args.nodes * args.gpus_per_node
    torch.cuda.set_device(local)
    pb = problem(args.nodes, args.gpus_per_node, steps=args.steps)
    box = [ts.nccl_unique_id() if rank == 0 else None]
    td.broadcast_object_list(box, src=0)
    table = ts.Table(n_rows=pb["n"], dim=pb["dim"], dp_cut=pb["dp_cut"], flex_cut=pb["flex_cut"],
                     tier_dest=pb["dest"], num_nodes=args.nodes, gpus_per_node=args.gpus_per_node,
                     rank=rank, device=local, weight_seed=77, optimizer=args.optimizer, lr=args.lr,
                     max_occurrences=int(max(r[rank].size for r in pb["steps_rows"])),
                     nccl_unique_id=box[0])
    if args.steps > 1:
        if args.pipelined:
            losses = list(table.train_steps_host([r[rank] for r in pb["steps_rows"]]))
        else:
            losses = [table.train_step_host(r[rank]) for r in pb["steps_rows"]]
        out = np.zeros((0, pb["dim"]), np.float32)
        loss = np.array(losses)
    else:
        rows = pb["rows"][rank]
        d_rows = torch.from_numpy(rows.view(np.int32)).cuda()
        d_out = torch.empty((rows.size, pb["dim"]), dtype=torch.float32, device="cuda")
        table.forward(d_rows.data_ptr(), rows.size, d_out.data_ptr())
        table.synchronize()
        out = d_out.cpu().numpy().copy()
        loss = table.loss()
        table.backward(d_out.data_ptr())
    table.synchronize()
    counters = table.counters()
    # rows stored on this rank
    n, dp, fx = pb["n"], pb["dp_cut"], pb["flex_cut"]
    c = np.arange(n)
    mine = (c < dp) | ((c >= dp) & (c < fx) & (pb["slot"] == rank % args.gpus_per_node)) | \
           ((c >= fx) & (pb["owner"] == rank))
    stored = c[mine].astype(np.uint32)
    wts, st = table.read_rows(stored, with_state=True)
    np.savez(Path(args.out) / f"rank{rank}.npz", out=out, loss=loss, counters=counters,
             stored=stored, weights=wts, state=st, shard=np.array(table.shard_rows()))
    table.close()
    td.barrier()
    td.destroy_process_group()


if __name__ == "__main__":
    main()
