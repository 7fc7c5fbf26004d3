"""Rank worker for tests/test_gpu_multigpu.py.  Two transports run the same
rank body (one forward + backward of a U-rank sharded table through the
C-ABI, or several host-buffer steps):
  * main(): launched by torch.distributed.run, one process per GPU, NCCL
    communicators + CUDA-IPC peer memory; dumps rank<g>.npz;
  * run_inproc(): every rank a thread of the calling process over one
    ts_group (several ranks may share one GPU), returning the results."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def problem(n_nodes, w, seed=11, steps=1, varying=False, dim=64):
    """rows[g] is rank g's first batch; steps > 1 adds steps_rows[s][g] for
    the host-API multi-step case, batches growing step to step (so any
    per-step buffer sized by the batch would have to move).  varying: ragged
    batches instead -- every step a random size in [0, 6000) per rank, with
    empty batches on rank 0 at step 7 and on every rank at step 11."""
    import oracle_bind as orc
    u = n_nodes * w
    n = 12000
    dp_cut, flex_cut = 150, 1500 if n_nodes * w > 1 else 150
    rng = np.random.default_rng(seed)
    p = np.arange(1, n + 1, dtype=np.float64) ** -1.1
    occ = [int(x) for x in rng.integers(3000, 6000, size=u)]
    rows = [rng.choice(n, size=o, p=p / p.sum()).astype(np.uint32) for o in occ]
    steps_rows = [rows]
    for s in range(1, steps):
        if varying:
            sizes = [int(x) for x in rng.integers(0, 6000, size=u)]
            if s == 7:
                sizes[0] = 0
            if s == 11:
                sizes = [0] * u
        else:
            sizes = [o + 1500 * s for o in occ]
        steps_rows.append([rng.choice(n, size=o, p=p / p.sum()).astype(np.uint32) for o in sizes])
    tier, owner, slot = orc.assign_rows(np.zeros(n, np.uint32), np.arange(n, dtype=np.uint64),
                                        dp_cut, flex_cut, u, w, 2)
    dest = np.where(tier == 1, slot, owner).astype(np.uint8)
    return dict(n=n, dim=dim, dp_cut=dp_cut, flex_cut=flex_cut, rows=rows, tier=tier, owner=owner,
                slot=slot, dest=dest, steps_rows=steps_rows)


def rank_body(rank, nodes, w, optimizer, lr, steps, pipelined, device, recv_hint=0, varying=False, dim=64,
              **table_kw):
    """One rank's forward + backward (steps == 1, device buffers) or `steps`
    host-buffer steps, through the C-ABI; returns what the parent test
    checks.  table_kw carries the transport: nccl_unique_id (one process per
    rank) or group (in-process ranks)."""
    import torch
    import paper_2301_02959_b200 as ts

    torch.cuda.set_device(device)
    pb = problem(nodes, w, steps=steps, varying=varying, dim=dim)
    table = ts.Table(n_rows=pb["n"], dim=pb["dim"], dp_cut=pb["dp_cut"], flex_cut=pb["flex_cut"],
                     tier_dest=pb["dest"], num_nodes=nodes, gpus_per_node=w,
                     rank=rank, device=device, weight_seed=77, optimizer=optimizer, lr=lr,
                     max_occurrences=int(max(r[rank].size for r in pb["steps_rows"])),
                     recv_rows_hint=recv_hint, **table_kw)
    if steps > 1:
        if pipelined:
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
    table.synchronize()  # collective: every rank's replica stores have landed
    counters = table.counters()
    # rows stored on this rank
    n, dp, fx = pb["n"], pb["dp_cut"], pb["flex_cut"]
    c = np.arange(n)
    mine = (c < dp) | ((c >= dp) & (c < fx) & (pb["slot"] == rank % w)) | \
           ((c >= fx) & (pb["owner"] == rank))
    stored = c[mine].astype(np.uint32)
    wts, st = table.read_rows(stored, with_state=True)
    res = dict(out=out, loss=loss, counters=counters, stored=stored, weights=wts, state=st,
               shard=np.array(table.shard_rows()), recv_capacity=np.array(table.recv_capacity()))
    table.close()
    return res


def run_inproc(nodes, w, optimizer, lr, steps=1, pipelined=False, env=None, recv_hint=0, varying=False, dim=64):
    """All U ranks as threads of this process over one ts_group (rank g on
    GPU g % device_count, so several ranks share a GPU on a small box)."""
    import threading
    import paper_2301_02959_b200 as ts

    u = nodes * w
    ndev = max(1, ts.device_count())
    saved = {}
    for k, v in (env or {}).items():  # schedule knobs are read at table creation
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    grp = ts.Group(u)
    results, errors = [None] * u, [None] * u

    def body(g):
        try:
            results[g] = rank_body(g, nodes, w, optimizer, lr, steps, pipelined, g % ndev, recv_hint=recv_hint,
                                   varying=varying, dim=dim, group=grp)
        except BaseException as e:  # noqa: BLE001 - reported by the caller
            errors[g] = e
            grp.abort()  # the other ranks' collectives fail now, not at the timeout

    try:
        threads = [threading.Thread(target=body, args=(g,)) for g in range(u)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for g, e in enumerate(errors):
        if e is not None:
            raise RuntimeError(f"in-process rank {g} failed: {e!r}") from e
    grp.close()
    return results


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, required=True)
    ap.add_argument("--gpus-per-node", type=int, required=True)
    ap.add_argument("--optimizer", type=int, default=1)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--steps", type=int, default=1, help="> 1: host-buffer steps (train_step_host)")
    ap.add_argument("--pipelined", action="store_true", help="the steps in one train_steps_host call")
    ap.add_argument("--recv-hint", type=int, default=0, help="recv_rows_hint (tiny: forces regrowth)")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import torch.distributed as td
    import paper_2301_02959_b200 as ts

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo")
    assert world == args.nodes * args.gpus_per_node
    box = [ts.nccl_unique_id() if rank == 0 else None]
    td.broadcast_object_list(box, src=0)
    res = rank_body(rank, args.nodes, args.gpus_per_node, args.optimizer, args.lr, args.steps,
                    args.pipelined, local, recv_hint=args.recv_hint, nccl_unique_id=box[0])
    np.savez(Path(args.out) / f"rank{rank}.npz", **res)
    td.barrier()
    td.destroy_process_group()


if __name__ == "__main__":
    main()
