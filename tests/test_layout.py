"""Host logic of the U > 1 path, on the CPU: the shard layout every rank
derives from the planner's placement bytes, and the per-step all-to-allv plan
(including a gloo world-size-2 run where each process computes its own plan
from all-gathered counts and the pairs must agree)."""
import os
import socket

import numpy as np
import pytest

from paper_2301_02959_b200 import capi
import oracle_bind as orc


def make_dest(n, dp_cut, flex_cut, u, w, seed=3):
    tier, owner, slot = orc.assign_rows(np.zeros(n, np.uint32), np.arange(n, dtype=np.uint64),
                                        dp_cut, flex_cut, u, w, seed)
    return np.where(tier == 1, slot, owner).astype(np.uint8), tier, owner, slot


@pytest.mark.parametrize("n_nodes,w", [(1, 1), (1, 4), (2, 2), (2, 4), (4, 8)])
def test_shard_layout_partitions_rows(n_nodes, w):
    u = n_nodes * w
    n, dp_cut, flex_cut = 20000, 300, 2500
    dest, tier, owner, slot = make_dest(n, dp_cut, flex_cut, u, w)
    seen_rw = np.zeros(n, np.int32)
    for g in range(u):
        ids, (dp, fl, rw) = capi.shard_layout(n, dp_cut, flex_cut, dest, n_nodes, w, g)
        assert dp == dp_cut
        assert fl == int((slot[dp_cut:flex_cut] == g % w).sum())
        assert rw == int((owner[flex_cut:] == g).sum())
        mine = np.zeros(n, bool)
        mine[:dp_cut] = True
        mine[dp_cut:flex_cut] = slot[dp_cut:flex_cut] == g % w
        mine[flex_cut:] = owner[flex_cut:] == g
        local = np.sort(ids[mine])
        # the rows a rank stores map onto [0, local_rows) exactly once,
        # and each tier keeps canonical order inside the shard
        assert np.array_equal(local, np.arange(dp + fl + rw))
        for lo, hi in ((0, dp_cut), (dp_cut, flex_cut), (flex_cut, n)):
            sub = ids[lo:hi][mine[lo:hi]]
            assert np.all(np.diff(sub.astype(np.int64)) > 0)
        seen_rw[flex_cut:] += mine[flex_cut:]
    assert np.all(seen_rw[flex_cut:] == 1), "every RW row lives on exactly one rank"


def test_shard_layout_rejects_bad_bytes():
    dest = np.full(100, 9, np.uint8)
    with pytest.raises(capi.TSError) as e:
        capi.shard_layout(100, 10, 20, dest, 2, 2, 0)
    assert e.value.kind == "ValidationError"


def random_starts(rng, u, w):
    nb = u + w + 1
    counts = rng.integers(0, 50, size=(u, nb))
    starts = np.zeros((u, nb + 1), np.uint32)
    starts[:, 1:] = np.cumsum(counts, axis=1)
    return starts


@pytest.mark.parametrize("n_nodes,w", [(1, 2), (2, 2), (2, 4), (1, 8)])
def test_exchange_plan_pairwise_consistent(n_nodes, w):
    rng = np.random.default_rng(n_nodes * 10 + w)
    u = n_nodes * w
    starts = random_starts(rng, u, w)
    plans = [capi.exchange_plan(n_nodes, w, g, starts) for g in range(u)]
    for p in range(u):
        for q in range(u):
            if p == q:
                continue
            # RW part p -> q and Flex part p -> q (same node only)
            assert plans[p]["send_cnt"][2 * q] == plans[q]["recv_cnt"][2 * p]
            assert plans[p]["send_cnt"][2 * q + 1] == plans[q]["recv_cnt"][2 * p + 1]
            if p // w != q // w:
                assert plans[p]["send_cnt"][2 * q + 1] == 0
    for g, x in enumerate(plans):
        assert x["recv_total"] == int(x["recv_cnt"].sum())
        # receive buffer ordered by source rank, contiguous, no overlap
        order = [(x["recv_off"][i], x["recv_cnt"][i]) for i in range(2 * u) if x["recv_cnt"][i]]
        pos = 0
        for off, cnt in order:
            assert off == pos
            pos += cnt
        before = sum(int(x["recv_cnt"][2 * p] + x["recv_cnt"][2 * p + 1]) for p in range(g))
        assert x["recv_before"] == before


def _gloo_worker(rank, world, port, w, q):
    import torch
    import torch.distributed as td
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_nodes = world // w
        u = world
        rng = np.random.default_rng(100 + rank)
        nb = u + w + 1
        counts = rng.integers(0, 1000, size=nb)
        mine = np.zeros(nb + 1, np.uint32)
        mine[1:] = np.cumsum(counts)
        # the same all-gather the table does over NCCL, here over gloo
        t = torch.from_numpy(mine.astype(np.int64))
        bufs = [torch.zeros_like(t) for _ in range(world)]
        td.all_gather(bufs, t)
        starts = np.stack([b.numpy() for b in bufs]).astype(np.uint32)
        plan = capi.exchange_plan(n_nodes, w, rank, starts)
        # exchange my send counts to the peer and compare with its recv plan
        send = torch.from_numpy(plan["send_cnt"].astype(np.int64))
        recv = torch.from_numpy(plan["recv_cnt"].astype(np.int64))
        all_send = [torch.zeros_like(send) for _ in range(world)]
        td.all_gather(all_send, send)
        ok = True
        for p in range(world):
            if p == rank:
                continue
            ok &= int(all_send[p][2 * rank]) == int(recv[2 * p])
            ok &= int(all_send[p][2 * rank + 1]) == int(recv[2 * p + 1])
        q.put((rank, ok))
    finally:
        td.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,w", [(2, 2), (2, 1)])
def test_exchange_plan_gloo_world(world, w):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, w, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(results.values()), results
