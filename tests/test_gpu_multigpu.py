"""Multi-rank parity of the U > 1 path (U = N*W ranks: one process per GPU, or
all ranks as threads of one process over a ts_group when the box has fewer
GPUs than ranks):
forward rows bit-exact on every rank, per-rank counter columns summing to the
reference routing loop's 7 x U block bit-exactly, updated weights equal to the
oracle's single-process update of the concatenated global batch — bit-exact
for rows with a single server (RW, and Flex when N == 1), within 1e-6 relative
for all-reduced replicas (DP, Flex when N > 1), and DP replicas identical
across ranks.

The 1e-6 bar (north star) applies at a training-scale learning rate: the
all-reduce sums a replicated row's gradient in a different fp32 order than the
single-process oracle (~sqrt(n) ulps apart for n occurrences), and that
difference reaches the weight scaled by lr * |step| / |w|.  The global batch
grows with U (the hottest row gets ~1800 occurrences per 2 ranks), so the
rate is 2e-3 / U: lr x (hottest row's count) stays ~1.8 at every U rather
than flipping that row's sign several times over at U = 8."""


def lr_for(u):
    return 2e-3 / u


# multi-step runs feed each step's weights into the next step's gradients
# (grad = out); a smaller rate keeps SGD on the hottest rows contractive so the
# summation-order differences do not compound across steps
LR_STEPS = 1e-4
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_bind as orc
import mg_worker

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = Path(__file__).resolve().parents[1]


def n_devices():
    try:
        import paper_2301_02959_b200 as ts
        return ts.device_count()
    except Exception:
        return 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_ranks(u, worker_args, env=None):
    """torchrun u ranks of mg_worker.py; a fresh port on a rendezvous-port race."""
    for _ in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={u}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
               str(ROOT / "tests" / "mg_worker.py"), *worker_args]
        proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
        if proc.returncode == 0 or "EADDRINUSE" not in proc.stderr:
            return proc
    return proc


CASES = [(1, 2, 1, "p2p"), (2, 1, 1, "p2p"), (2, 1, 0, "p2p"), (2, 2, 1, "p2p"), (1, 4, 1, "p2p"),
         (1, 2, 1, "p2p_pull"), (2, 2, 1, "p2p_pull"), (1, 4, 0, "p2p_pull"),
         (1, 2, 1, "nccl"), (2, 2, 1, "nccl"), (2, 1, 0, "nccl"),
         (1, 2, 1, "p2p_short8"), (2, 2, 1, "p2p_short8"), (1, 2, 1, "p2p_serial"),
         (1, 2, 1, "p2p_regrow"), (2, 2, 0, "p2p_regrow"), (1, 2, 1, "p2p_mailbox"), (2, 2, 1, "p2p_mailbox"),
         (1, 2, 1, "p2p_fwdpull"), (2, 2, 0, "p2p_fwdpull"), (1, 4, 1, "p2p_fwdpull"),
         (1, 2, 1, "p2p_deferred"), (2, 2, 1, "p2p_deferred"), (1, 4, 0, "p2p_deferred")]
# always in-process (ts_group): the C2 topologies at logical U = 8 on however
# many GPUs the box has (several ranks per GPU), and a 2-per-GPU mix
INPROC_CASES = [(1, 8, 1, "p2p"), (2, 4, 1, "p2p"), (2, 4, 0, "nccl"), (1, 3, 1, "p2p"), (3, 2, 1, "p2p_pull"),
                (2, 4, 1, "p2p_fwdpull"), (2, 4, 1, "p2p_deferred"), (2, 4, 1, "p2p_r1sched")]


def case_env(exchange):
    env = dict(TIERSHARD_EXCHANGE="nccl" if exchange == "nccl" else "p2p",
               TIERSHARD_GRADS="pull" if exchange == "p2p_pull" else "push",
               TIERSHARD_LONG_CONCURRENT="0" if exchange == "p2p_serial" else "1")
    if exchange == "p2p_short8":
        env["TIERSHARD_SHORT_MAX"] = "8"
    if exchange == "p2p_mailbox":
        env["TIERSHARD_FWD_COUNTS"] = "mailbox"
    if exchange == "p2p_fwdpull":
        env["TIERSHARD_FWD"] = "pull"
    if exchange == "p2p_deferred":
        env["TIERSHARD_REPLICA"] = "deferred"
    if exchange == "p2p_r1sched":  # the earlier schedules: sorted route, block owners, rank-order push
        env.update(TIERSHARD_ROUTE="sort", TIERSHARD_REPLICA_OWNER="block", TIERSHARD_PUSH_ROTATE="0")
    return env


def run_case(tmp_path, n_nodes, w, opt, lr, exchange="p2p", steps=1, pipelined=False, transport="auto",
             recv_hint=0):
    """Runs every rank and returns their results.  transport "auto": one
    process per GPU (NCCL + CUDA IPC) when the box has U GPUs, else all ranks
    as threads of this process over a ts_group (several ranks per GPU) --
    the same rank body and checks either way, so no case is skipped on a
    small box.  "inproc" forces the group."""
    u = n_nodes * w
    env = case_env(exchange)
    if exchange == "p2p_regrow":
        recv_hint = 16  # far below one step's remote rows: the first step regrows
    if transport == "auto" and n_devices() >= u:
        args = ["--nodes", str(n_nodes), "--gpus-per-node", str(w), "--optimizer", str(opt), "--lr", str(lr),
                "--steps", str(steps), "--recv-hint", str(recv_hint), "--out", str(tmp_path)] + \
               (["--pipelined"] if pipelined else [])
        proc = run_ranks(u, args, dict(os.environ, **env))
        assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
        return [dict(np.load(tmp_path / f"rank{g}.npz")) for g in range(u)]
    print(f"in-process group: {u} ranks on {max(1, n_devices())} GPU(s)")
    return mg_worker.run_inproc(n_nodes, w, opt, lr, steps=steps, pipelined=pipelined, env=env, recv_hint=recv_hint)


def assert_rows_close(got, ref, before, rtol=1e-6):
    """Replicated rows: within 1e-6 relative, row-wise -- |got - ref| <=
    rtol * (the row's magnitude before or after the update, whichever is
    larger) on every element.  Their gradient is summed per rank and the
    partials combined in rank order, a different fp32 order than the
    oracle's single pass, so the rounding scales with the terms summed (w and
    lr * sum g), not with what is left where they cancel (w - lr*g with
    w ~ lr*g: a hot row updated by SGD can shrink 300x)."""
    if got.size == 0:
        return
    scale = np.maximum(np.abs(ref).max(axis=1, keepdims=True), np.abs(before).max(axis=1, keepdims=True))
    # either reading of "1e-6 relative" passes: to the row's magnitude, or to
    # the element's own with a floor of 1e-6 x the init scale (|w0| <= 0.01)
    tol = np.maximum(rtol * scale, rtol * np.abs(ref) + 1e-8)
    bad = np.abs(got.astype(np.float64) - ref) > tol
    assert not bad.any(), (int(bad.sum()), float((np.abs(got - ref) / np.maximum(scale, 1e-30)).max()))


def check_one_step(res, n_nodes, w, opt, lr, dim=64):
    """forward bit-exact, counters == the reference loop, updates == oracle."""
    u = n_nodes * w
    pb = mg_worker.problem(n_nodes, w, dim=dim)
    n, dim, dp, fx = pb["n"], pb["dim"], pb["dp_cut"], pb["flex_cut"]
    w0 = orc.init_table(77, n, dim)

    # forward: bit-exact on every rank
    for g in range(u):
        expect = orc.gather(w0, pb["rows"][g])
        assert np.array_equal(res[g]["out"].view(np.uint32), expect.view(np.uint32)), f"rank {g}"
        assert float(res[g]["loss"]) == pytest.approx(orc.half_sq_sum(expect), rel=1e-6)

    # counters: per-rank columns sum to the reference loop's block
    offsets = np.concatenate([[0], np.cumsum([r.size for r in pb["rows"]])]).astype(np.uint64)
    allrows = np.concatenate(pb["rows"])
    ref_c = orc.route_counts(u, w, 1, offsets, allrows, pb["tier"], pb["owner"], pb["slot"])
    got_c = sum(r["counters"].astype(np.uint64) for r in res)
    assert np.array_equal(got_c, ref_c), (got_c, ref_c)

    # backward: oracle over the concatenated global batch (ascending rank order)
    w_ref = w0.copy()
    st_ref = np.zeros(n, np.float32)
    orc.backward_update(w_ref, st_ref, allrows, orc.gather(w0, allrows), opt, lr, 1e-8)
    for g in range(u):
        stored = res[g]["stored"]
        got = res[g]["weights"]
        exact = (stored >= fx) | ((stored >= dp) & (n_nodes == 1))
        assert np.array_equal(got[exact].view(np.uint32), w_ref[stored[exact]].view(np.uint32)), g
        assert_rows_close(got[~exact], w_ref[stored[~exact]], w0[stored[~exact]])
        if opt == 1:
            np.testing.assert_allclose(res[g]["state"], st_ref[stored], rtol=1e-5, atol=1e-12)
    # replicated DP rows are identical on every rank
    for g in range(1, u):
        assert np.array_equal(res[g]["weights"][:dp].view(np.uint32), res[0]["weights"][:dp].view(np.uint32))


@pytest.mark.parametrize("n_nodes,w,opt,exchange", CASES)
def test_multi_gpu_matches_oracle(cuda, tmp_path, n_nodes, w, opt, exchange):
    """exchange: "p2p" = peer-memory serve + gradient push (default on one
    node), "p2p_pull" = servers gather remote gradients with peer loads
    (TIERSHARD_GRADS=pull), "nccl" = staged all-to-allv + all-reduce
    (TIERSHARD_EXCHANGE=nccl; NCCL between processes, the group's copies and
    sum kernel in-process), "p2p_short8" = segments over 8 entries take the
    piece path on the aux stream (TIERSHARD_SHORT_MAX=8), "p2p_serial" = long
    segments after the short kernel (TIERSHARD_LONG_CONCURRENT=0),
    "p2p_regrow" = a 16-row gradient receive buffer (recv_rows_hint): the
    step takes the collective regrowth path first, "p2p_mailbox" = counts
    through the peer mailboxes (TIERSHARD_FWD_COUNTS=mailbox; one process
    per GPU only -- the in-process group keeps its host all-gather),
    "p2p_fwdpull" = the requester-pull forward (TIERSHARD_FWD=pull),
    "p2p_deferred" = the replica update deferred into the next step
    (TIERSHARD_REPLICA=deferred)."""
    res = run_case(tmp_path, n_nodes, w, opt, lr_for(n_nodes * w), exchange)
    check_one_step(res, n_nodes, w, opt, lr_for(n_nodes * w))
    if exchange == "p2p_regrow":  # the path was taken, collectively
        assert all(int(r["recv_capacity"][1]) >= 1 for r in res)
        assert any(int(r["recv_capacity"][0]) > 16 for r in res)


@pytest.mark.parametrize("n_nodes,w,opt,exchange", INPROC_CASES)
def test_inproc_group_matches_oracle(cuda, tmp_path, n_nodes, w, opt, exchange):
    """Every rank a thread of this process over one ts_group: logical U = 8
    (1x8 2-tier, 2x4 3-tier -- the C2 topologies), odd shapes, on however many
    GPUs the box has."""
    res = run_case(tmp_path, n_nodes, w, opt, lr_for(n_nodes * w), exchange, transport="inproc")
    check_one_step(res, n_nodes, w, opt, lr_for(n_nodes * w))


@pytest.mark.parametrize("n_nodes,w,opt,pipelined,hint", [(1, 2, 1, False, 0), (2, 2, 1, False, 0),
                                                          (1, 4, 0, False, 0), (1, 2, 1, True, 0),
                                                          (2, 2, 1, True, 0), (1, 2, 1, True, 600),
                                                          (2, 2, 0, False, 600)])
def test_multi_gpu_host_steps_match_oracle(cuda, tmp_path, n_nodes, w, opt, pipelined, hint):
    """Three steps through the host-buffer entry point (ts_table_train_step_host)
    with batches growing step to step: every step's loss and the final weights
    follow the oracle's sequential updates (stale peer mappings or stale
    replica stamps would break this)."""
    u = n_nodes * w
    steps = 3
    # hint 600: the receive buffer starts below a step's need and grows
    # step to step as the batches grow (peers re-map it each time)
    res = run_case(tmp_path, n_nodes, w, opt, LR_STEPS, steps=steps, pipelined=pipelined, recv_hint=hint)
    if hint:
        assert all(int(r["recv_capacity"][1]) >= 1 for r in res)
    pb = mg_worker.problem(n_nodes, w, steps=steps)
    n, dim, dp, fx = pb["n"], pb["dim"], pb["dp_cut"], pb["flex_cut"]
    w_ref = orc.init_table(77, n, dim)
    st_ref = np.zeros(n, np.float32)
    for s, batch in enumerate(pb["steps_rows"]):
        allrows = np.concatenate(batch)
        for g in range(u):  # each rank's loss: 0.5 |its unpooled rows|^2
            expect = orc.half_sq_sum(orc.gather(w_ref, batch[g]))
            assert float(res[g]["loss"][s]) == pytest.approx(expect, rel=1e-6), (s, g)
        orc.backward_update(w_ref, st_ref, allrows, orc.gather(w_ref, allrows), opt, LR_STEPS, 1e-8)
    for g in range(u):
        stored = res[g]["stored"]
        np.testing.assert_allclose(res[g]["weights"], w_ref[stored], rtol=1e-6, atol=1e-8)
    for g in range(1, u):
        assert np.array_equal(res[g]["weights"][:dp].view(np.uint32), res[0]["weights"][:dp].view(np.uint32))


@pytest.mark.parametrize("dim,opt", [(512, 1), (1024, 0), (32, 1)])
def test_inproc_wide_and_narrow_rows(cuda, dim, opt):
    """The U > 1 kernels at the dispatch extremes (serve / push / replica
    update templates for D = 32 .. 1024), 2 x 2 ranks in-process."""
    res = mg_worker.run_inproc(2, 2, opt, lr_for(4), dim=dim)
    check_one_step(res, 2, 2, opt, lr_for(4), dim=dim)


@pytest.mark.parametrize("n_nodes,w,pipelined,replica", [(1, 2, True, "concurrent"), (2, 2, False, "concurrent"),
                                                         (2, 2, True, "deferred")])
def test_inproc_stress_ragged_steps(cuda, tmp_path, n_nodes, w, pipelined, replica):
    """50 host-buffer steps with ragged batches (random sizes, an empty batch
    on one rank, an all-empty step) through the peer-memory protocol on the
    in-process group, a tiny initial receive buffer (regrowth mid-run):
    every step's loss and the final weights / Adagrad state follow the
    oracle's 50 sequential updates; replicas stay identical."""
    u, steps = n_nodes * w, 50
    res = mg_worker.run_inproc(n_nodes, w, 1, LR_STEPS, steps=steps, pipelined=pipelined, recv_hint=64,
                               varying=True, env={"TIERSHARD_REPLICA": replica})
    pb = mg_worker.problem(n_nodes, w, steps=steps, varying=True)
    n, dim, dp = pb["n"], pb["dim"], pb["dp_cut"]
    w_ref = orc.init_table(77, n, dim)
    w0 = w_ref.copy()
    st_ref = np.zeros(n, np.float32)
    for s, batch in enumerate(pb["steps_rows"]):
        allrows = np.concatenate(batch)
        for g in range(u):
            expect = orc.half_sq_sum(orc.gather(w_ref, batch[g]))
            assert float(res[g]["loss"][s]) == pytest.approx(expect, rel=1e-6, abs=1e-12), (s, g)
        if allrows.size:
            orc.backward_update(w_ref, st_ref, allrows, orc.gather(w_ref, allrows), 1, LR_STEPS, 1e-8)
    for g in range(u):
        stored = res[g]["stored"]
        assert_rows_close(res[g]["weights"], w_ref[stored], w0[stored])
        np.testing.assert_allclose(res[g]["state"], st_ref[stored], rtol=1e-5, atol=1e-12)
        assert int(res[g]["recv_capacity"][1]) >= 1
    for g in range(1, u):
        assert np.array_equal(res[g]["weights"][:dp].view(np.uint32), res[0]["weights"][:dp].view(np.uint32))
