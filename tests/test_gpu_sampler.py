"""GPU workload sampler (ts_sampler_*).

Statistical, not bit-wise, equivalence with the host Workload: every sample is
the reference's per-sample procedure (Poisson(L) length, alias draws over the
same AliasTable) on its own stream.  Checked here:
  * sample lengths: mean and variance of Poisson(L), both PTRD (L >= 10) and
    multiplication (L < 10) regimes;
  * row frequencies: E[count_i] = p_i * samples (p sums to L), z-tests on the
    hottest rows and a chi-square over the top 200;
  * the same law as the host Workload (bit-exact reference sampler) on the
    same distribution: mean occurrences and hot-row shares agree;
  * per-sample streams make sharding exact: samples [0, 2S) in one call equal
    [0, S) + [S, 2S) in two (a U-GPU job samples each rank's block locally);
  * determinism, iteration independence, capacity errors.
"""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from specs import TS_DRIVER

pytestmark = pytest.mark.gpu


def export(tmp: Path, rows: int, exponent: float, length: float, batch: int = 64, iters: int = 2):
    spec = dict(tables=[dict(table_id=0, rows=rows, exponent=exponent, target_length=length, seed=5)],
                topology=dict(num_nodes=1, gpus_per_node=1, a2a_global_gibs=1, a2a_intra_gibs=1,
                              ar_global_gibs=1, ar_cross_gibs=1),
                cost_model=dict(local_batch=batch, embedding_dim=32), goal="rw", frontier=False,
                hash_seed=2, workload=dict(seed=7, iterations=iters), export_dir=str(tmp), export_alias=True)
    (tmp / "spec.json").write_text(json.dumps(spec))
    subprocess.run([str(TS_DRIVER), str(tmp / "spec.json"), str(tmp / "doc.json")], check=True, timeout=300)
    doc = json.loads((tmp / "doc.json").read_text())
    prob = np.fromfile(tmp / "alias.prob.f64", np.float64)
    idx = np.fromfile(tmp / "alias.idx.u32", np.uint32)
    return doc, prob, idx


def run(sampler, it, begin, samples, cap):
    import torch
    rows = torch.empty(cap, dtype=torch.int32, device="cuda")
    offs = torch.empty(samples + 1, dtype=torch.int64, device="cuda")
    occ = sampler.iteration(it, begin, samples, rows.data_ptr(), cap, offs.data_ptr())
    torch.cuda.synchronize()
    return rows[:occ].cpu().numpy().view(np.uint32), offs.cpu().numpy().astype(np.uint64)


@pytest.mark.parametrize("length", [40.0, 3.0])
def test_lengths_and_row_frequencies(cuda, tmp_path, length):
    import paper_2301_02959_b200 as ts
    doc, prob, idx = export(tmp_path, rows=20000, exponent=1.05, length=length)
    L = float(doc["expected_length"])
    assert L == pytest.approx(length, rel=1e-9)
    s = ts.Sampler(prob, idx, L, seed=123)
    S = 40000
    rows, offs = run(s, 0, 0, S, int(S * L * 1.5) + 1024)
    counts = np.diff(offs.astype(np.int64))
    assert offs[0] == 0 and offs[-1] == rows.size
    # Poisson(L): mean within 5 sigma, variance within 5 %
    assert abs(counts.mean() - L) < 5 * np.sqrt(L / S)
    assert counts.var() == pytest.approx(L, rel=0.05)
    # row law: alias table -> exact category probabilities q_i (sum 1)
    n = prob.size
    q = prob / n
    np.add.at(q, idx, (1.0 - prob) / n)
    freq = np.bincount(rows, minlength=n).astype(np.float64)
    exp = q * rows.size
    top = np.argsort(-q)[:200]
    z = (freq[top] - exp[top]) / np.sqrt(exp[top])
    assert np.abs(z).max() < 6, np.abs(z).max()
    chi2 = float((z ** 2).sum())
    from scipy.stats import chi2 as c2
    assert chi2 < c2.ppf(0.9999, df=199)
    s.close()


def test_matches_host_workload_law(cuda, tmp_path):
    """Same distribution, host Workload (bit-exact reference sampler) vs GPU:
    mean occurrences per sample and the hottest rows' shares agree."""
    import paper_2301_02959_b200 as ts
    doc, prob, idx = export(tmp_path, rows=50000, exponent=1.1, length=64.0, batch=512, iters=8)
    host = np.concatenate([np.fromfile(tmp_path / f"batch_{i}.rows.u32", np.uint32) for i in range(8)])
    host_samples = 8 * 512
    s = ts.Sampler(prob, idx, float(doc["expected_length"]), seed=99)
    dev, _ = run(s, 0, 0, host_samples, host_samples * 128)
    assert abs(dev.size / host_samples - host.size / host_samples) < 5 * np.sqrt(64.0 / host_samples) * 1.5
    n = prob.size
    hf = np.bincount(host, minlength=n) / host.size
    df = np.bincount(dev, minlength=n) / dev.size
    for r in range(10):  # canonical rows 0.. are the hottest
        assert df[r] == pytest.approx(hf[r], abs=5 * np.sqrt(hf[r] / dev.size) + 1e-4)
    s.close()


def test_sharding_determinism_and_errors(cuda, tmp_path):
    import paper_2301_02959_b200 as ts
    doc, prob, idx = export(tmp_path, rows=5000, exponent=1.0, length=20.0)
    L = float(doc["expected_length"])
    s = ts.Sampler(prob, idx, L, seed=1)
    cap = 4096 * 64
    a, ao = run(s, 3, 0, 4096, cap)
    b1, b1o = run(s, 3, 0, 2048, cap)
    b2, b2o = run(s, 3, 2048, 2048, cap)
    assert np.array_equal(a, np.concatenate([b1, b2]))
    again, _ = run(s, 3, 0, 4096, cap)
    assert np.array_equal(a, again)
    other, _ = run(s, 4, 0, 4096, cap)
    assert not np.array_equal(a[:1000], other[:1000])
    with pytest.raises(ts.TSError) as e:
        run(s, 3, 0, 4096, 100)
    assert e.value.kind == "ValidationError" and "capacity" in e.value.message
    s.close()
    with pytest.raises(ts.TSError) as e:
        ts.Sampler(prob, idx, 0.0, seed=1)
    assert e.value.kind == "ValidationError"
