"""Value-path parity on one GPU (U = 1): the CUDA lookup/update entry points
through the C-ABI against the CPU restatement in oracle/restate.c.

Bar: gather bit-exact; segment sums + SGD / row-wise Adagrad bit-exact (the
restatement fixes the fp32 summation order, see restate.h); loss (a reported
scalar, summed in a different order) within 1e-6 relative.
"""
import numpy as np
import pytest

import oracle_bind as orc

pytestmark = pytest.mark.gpu

SEED = 1234


def _torch():
    import torch
    return torch


def zipf_rows(rng, n, occ, s=1.05, hot=None):
    ranks = np.arange(1, n + 1, dtype=np.float64)
    p = ranks ** -s
    p /= p.sum()
    rows = rng.choice(n, size=occ, p=p).astype(np.uint32)
    if hot is not None:  # force very long segments (> 256 entries) on a few rows
        for r, count in hot:
            idx = rng.choice(occ, size=min(count, occ), replace=False)
            rows[idx] = r
    return rows


def run_step(table, rows, dim):
    torch = _torch()
    occ = rows.size
    d_rows = torch.from_numpy(rows.astype(np.int32)).cuda()
    d_out = torch.empty((max(occ, 1), dim), dtype=torch.float32, device="cuda")
    table.forward(d_rows.data_ptr(), occ, d_out.data_ptr())
    table.synchronize()
    out = d_out[:occ].cpu().numpy().copy()
    loss = table.loss()
    table.backward(d_out.data_ptr())
    table.synchronize()
    return out, loss


@pytest.mark.parametrize("dim", [32, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("optimizer", [orc.OPT_SGD, orc.OPT_ROWWISE_ADAGRAD])
def test_single_gpu_step_bit_exact(cuda, dim, optimizer):
    import paper_2301_02959_b200 as ts
    rng = np.random.default_rng(dim * 7 + optimizer)
    n, occ = 6000, 30000
    rows = zipf_rows(rng, n, occ, hot=[(3, 2000), (17, 700), (4000, 300)])
    lr, eps = 0.05, 1e-8
    table = ts.Table(n_rows=n, dim=dim, dp_cut=50, flex_cut=50, weight_seed=SEED,
                     optimizer=optimizer, lr=lr, eps=eps, max_occurrences=occ)
    out, loss = run_step(table, rows, dim)
    w = orc.init_table(SEED, n, dim)
    expect = orc.gather(w, rows)
    assert np.array_equal(out.view(np.uint32), expect.view(np.uint32)), "gather must be bit-exact"
    assert loss == pytest.approx(orc.half_sq_sum(expect), rel=1e-6)
    state = np.zeros(n, np.float32)
    nseg = orc.backward_update(w, state, rows, expect, optimizer, lr, eps)
    got, got_state = table.read_rows(np.arange(n, dtype=np.uint32), with_state=True)
    assert np.array_equal(got.view(np.uint32), w.view(np.uint32)), (
        f"max abs diff {np.abs(got - w).max()}")
    if optimizer == orc.OPT_ROWWISE_ADAGRAD:
        assert np.array_equal(got_state.view(np.uint32), state.view(np.uint32))
    c = table.counters()
    assert int(c[6, 0]) == nseg == len(np.unique(rows))
    assert int(c[5, 0]) == occ
    assert int(c[4, 0]) == int((rows < 50).sum())
    table.close()


def test_two_steps_and_host_entry(cuda):
    """Two consecutive steps (weights feed the next forward) + the host-buffer
    entry point used for the end-to-end number."""
    import paper_2301_02959_b200 as ts
    rng = np.random.default_rng(5)
    n, dim, occ = 3000, 128, 12000
    lr = 0.1
    table = ts.Table(n_rows=n, dim=dim, dp_cut=10, flex_cut=10, weight_seed=SEED,
                     optimizer=orc.OPT_ROWWISE_ADAGRAD, lr=lr, max_occurrences=occ)
    w = orc.init_table(SEED, n, dim)
    state = np.zeros(n, np.float32)
    for step in range(2):
        rows = zipf_rows(rng, n, occ)
        loss = table.train_step_host(rows)
        expect = orc.gather(w, rows)
        assert loss == pytest.approx(orc.half_sq_sum(expect), rel=1e-6)
        orc.backward_update(w, state, rows, expect, orc.OPT_ROWWISE_ADAGRAD, lr, 1e-8)
    got = table.read_rows(np.arange(n, dtype=np.uint32))
    assert np.array_equal(got.view(np.uint32), w.view(np.uint32))


def test_pipelined_host_steps_match_oracle(cuda):
    """ts_table_train_steps_host: five steps (different sizes, one empty) in one
    pipelined call -- every loss and the final weights bit-exact with the
    oracle's sequential steps."""
    import paper_2301_02959_b200 as ts
    rng = np.random.default_rng(11)
    n, dim = 4000, 64
    sizes = [9000, 12000, 0, 7000, 12000]
    lr = 0.05
    table = ts.Table(n_rows=n, dim=dim, dp_cut=0, flex_cut=0, weight_seed=SEED,
                     optimizer=orc.OPT_ROWWISE_ADAGRAD, lr=lr, max_occurrences=max(sizes))
    batches = [zipf_rows(rng, n, k) if k else np.zeros(0, np.uint32) for k in sizes]
    losses = table.train_steps_host(batches)
    w = orc.init_table(SEED, n, dim)
    state = np.zeros(n, np.float32)
    for b, loss in zip(batches, losses):
        expect = orc.gather(w, b) if b.size else np.zeros((0, dim), np.float32)
        assert loss == pytest.approx(orc.half_sq_sum(expect), rel=1e-6, abs=1e-12)
        if b.size:
            orc.backward_update(w, state, b, expect, orc.OPT_ROWWISE_ADAGRAD, lr, 1e-8)
    got = table.read_rows(np.arange(n, dtype=np.uint32))
    assert np.array_equal(got.view(np.uint32), w.view(np.uint32))
    with pytest.raises(ts.TSError) as e:
        table.train_steps_host([np.zeros(max(sizes) + 1, np.uint32)])
    assert e.value.kind == "ValidationError"


def test_edge_cases(cuda):
    import paper_2301_02959_b200 as ts
    n, dim = 1000, 64
    table = ts.Table(n_rows=n, dim=dim, dp_cut=0, flex_cut=0, weight_seed=SEED, max_occurrences=5000)
    # empty batch: no-op
    assert table.train_step_host(np.zeros(0, np.uint32)) == 0.0
    # single occurrence, and the last row
    w = orc.init_table(SEED, n, dim)
    rows = np.array([n - 1], np.uint32)
    loss = table.train_step_host(rows)
    assert loss == pytest.approx(orc.half_sq_sum(w[n - 1:]), rel=1e-6)
    orc.backward_update(w, None, rows, w[n - 1:].copy(), orc.OPT_SGD, 0.01)
    assert np.array_equal(table.read_rows(rows).view(np.uint32), w[n - 1:].view(np.uint32))
    # one row repeated: a single very long segment (many pieces)
    rows = np.full(4999, 7, np.uint32)
    table.train_step_host(rows)
    w7 = w[7:8].copy()
    orc.backward_update(w, None, rows, np.repeat(w7, 4999, axis=0), orc.OPT_SGD, 0.01)
    assert np.array_equal(table.read_rows(np.array([7], np.uint32)).view(np.uint32),
                          w[7:8].view(np.uint32))
    # out-of-capacity batch and out-of-range rows are rejected loudly
    with pytest.raises(ts.TSError) as e:
        table.train_step_host(np.zeros(6000, np.uint32))
    assert e.value.kind == "ValidationError"
    with pytest.raises(ts.TSError):
        table.read_rows(np.array([n], np.uint32))


def test_bad_config_rejected(cuda):
    import paper_2301_02959_b200 as ts
    with pytest.raises(ts.TSError) as e:
        ts.Table(n_rows=100, dim=48, dp_cut=0, flex_cut=0)
    assert e.value.kind == "ConfigError"
    with pytest.raises(ts.TSError) as e:
        ts.Table(n_rows=100, dim=64, dp_cut=50, flex_cut=10)
    assert e.value.kind == "ValidationError"


@pytest.mark.parametrize("schedule", [
    {"TIERSHARD_LONG_CONCURRENT": "1"},
    {"TIERSHARD_LONG_CONCURRENT": "0"},
    {"TIERSHARD_LONG_CONCURRENT": "1", "TIERSHARD_SHORT_MAX": "8"},
    {"TIERSHARD_LONG_CONCURRENT": "1", "TIERSHARD_SHORT_MAX": "256"},
    {"TIERSHARD_DEDUP_IN_FORWARD": "0"},  # no aux stream: everything serial
])
def test_segment_schedules_bit_exact(cuda, monkeypatch, schedule):
    """Every segment schedule (long segments beside the short kernel on the aux
    stream or after it, the short/long threshold, dedup in the forward or the
    backward) gives the oracle's weights bit for bit over three steps."""
    import paper_2301_02959_b200 as ts
    for k, v in schedule.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(21)
    n, dim, occ = 5000, 128, 20000
    lr = 0.05
    table = ts.Table(n_rows=n, dim=dim, dp_cut=0, flex_cut=0, weight_seed=SEED,
                     optimizer=orc.OPT_ROWWISE_ADAGRAD, lr=lr, max_occurrences=occ)
    w = orc.init_table(SEED, n, dim)
    state = np.zeros(n, np.float32)
    for step in range(3):
        rows = zipf_rows(rng, n, occ, hot=[(1, 3000), (9, 600), (2500, 40)])
        loss = table.train_step_host(rows)
        expect = orc.gather(w, rows)
        assert loss == pytest.approx(orc.half_sq_sum(expect), rel=1e-6)
        orc.backward_update(w, state, rows, expect, orc.OPT_ROWWISE_ADAGRAD, lr, 1e-8)
    got, got_state = table.read_rows(np.arange(n, dtype=np.uint32), with_state=True)
    assert np.array_equal(got.view(np.uint32), w.view(np.uint32))
    assert np.array_equal(got_state.view(np.uint32), state.view(np.uint32))
    table.close()


@pytest.mark.parametrize("graph,lookahead", [("1", "0"), ("0", "0"), ("0", "1"), ("1", "1")])
def test_train_steps_graph_bit_exact(cuda, monkeypatch, graph, lookahead):
    """ts_table_train_step(s)_host at U = 1 with the step captured into a CUDA
    graph (TIERSHARD_GRAPH=1: re-captured every call and updated in place,
    re-instantiated when the topology changes -- e.g. an empty batch) and
    without: every step's loss and the final weights + state are the
    oracle's sequential updates, bit for bit."""
    import paper_2301_02959_b200 as ts
    monkeypatch.setenv("TIERSHARD_GRAPH", graph)
    monkeypatch.setenv("TIERSHARD_LOOKAHEAD", lookahead)  # cross-step dedup in train_steps_host
    n, dim, lr = 30_000, 128, 0.02
    rng = np.random.default_rng(12)
    sizes = [20_000, 23_000, 0, 17_000, 23_000]
    batches = [zipf_rows(rng, n, s) if s else np.zeros(0, np.uint32) for s in sizes]
    table = ts.Table(n_rows=n, dim=dim, dp_cut=200, flex_cut=200, weight_seed=SEED,
                     optimizer=ts.OPT_ROWWISE_ADAGRAD, lr=lr, max_occurrences=max(sizes))
    losses = list(table.train_steps_host(batches[:3])) + [table.train_step_host(b) for b in batches[3:]]
    w = orc.init_table(SEED, n, dim)
    st = np.zeros(n, np.float32)
    for s, b in enumerate(batches):
        out = orc.gather(w, b)
        assert losses[s] == pytest.approx(orc.half_sq_sum(out), rel=1e-6, abs=1e-12), s
        if b.size:
            orc.backward_update(w, st, b, out, orc.OPT_ROWWISE_ADAGRAD, lr, 1e-8)
    table.synchronize()
    got_w, got_s = table.read_rows(np.arange(n, dtype=np.uint32), with_state=True)
    assert np.array_equal(got_w.view(np.uint32), w.view(np.uint32))
    assert np.array_equal(got_s.view(np.uint32), st.view(np.uint32))
    table.close()
