"""Plan import from the reference's on-disk formats
and the raw-key device path.

CPU: the plan document + assignment CSV written by the reference's json_io
(oracle/_ref/ref_artifacts, or our byte-identical ts_artifacts where the
reference build is absent) are loaded by load_device_plan (bin/ts_plan_import);
the derived canonical keys and placement bytes must equal the oracle's
assign_rows restatement (restate.c) of the same rows, and every way the two
files can disagree is rejected with the reference's error classes.

GPU: the key map (ts_keymap_*) against a Python dict, and forward_keys
against forward on the canonical ids (bit-exact outputs and updates).
"""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_bind as orc
import test_io_parity as io

ROOT = Path(__file__).resolve().parents[1]
IMPORT = ROOT / "paper_2301_02959_b200" / "bin" / "ts_plan_import"
EXAMPLE = ROOT / "paper_2301_02959_b200" / "bin" / "ts_example"


def artifacts(tmp_path: Path, name: str) -> Path:
    """plan.json + assignment.csv for one of test_io_parity's manifests."""
    manifest = io.write_case(tmp_path / name / "in", *io.CASES[name], sim=False)
    exe = io.REF_ARTIFACTS if io.REF_ARTIFACTS.exists() else io.TS_ARTIFACTS
    out = tmp_path / name / "art"
    code, files = io.run_artifacts(exe, manifest, out)
    assert code == 0, files.get("error.txt")
    return out


def run_import(plan: Path, csv: Path, out: Path):
    proc = subprocess.run([str(IMPORT), str(plan), str(csv), str(out)], capture_output=True, timeout=300)
    err = (out / "error.txt").read_text() if (out / "error.txt").exists() else None
    return proc.returncode, err


def load_import(out: Path):
    s = json.loads((out / "summary.json").read_text())
    t = np.fromfile(out / "table.u32", np.uint32)
    r = np.fromfile(out / "row.u64", np.uint64)
    p = np.fromfile(out / "placement.u8", np.uint8)
    return s, t, r, p


def read_assignment(csv: Path):
    lines = csv.read_text().splitlines()[1:]
    t = np.array([int(x.split(",")[0]) for x in lines], np.uint32)
    r = np.array([int(x.split(",")[1]) for x in lines], np.uint64)
    return t, r, [x.split(",")[2] for x in lines]


@pytest.mark.parametrize("name", sorted(io.CASES))
def test_import_matches_oracle_placement(name, tmp_path):
    art = artifacts(tmp_path, name)
    code, err = run_import(art / "plan.json", art / "assignment.csv", tmp_path / "imp")
    assert code == 0, err
    s, t, r, p = load_import(tmp_path / "imp")
    doc = json.loads((art / "plan.json").read_text())
    assert (s["dp_cut"], s["flex_cut"], s["rows"]) == (doc["dp_cut"], doc["flex_cut"], doc["total_rows"])
    ct, cr, tiers = read_assignment(art / "assignment.csv")
    assert np.array_equal(t, ct) and np.array_equal(r, cr)
    u = doc["topology"]["num_nodes"] * doc["topology"]["gpus_per_node"]
    w = doc["topology"]["gpus_per_node"]
    tier, owner, slot = orc.assign_rows(t, r, doc["dp_cut"], doc["flex_cut"], u, w, doc["hash_seed"])
    expect = np.where(tier == 0, 0, np.where(tier == 1, slot, owner)).astype(np.uint8)
    assert np.array_equal(p, expect)
    assert [("dp", "flex", "rw")[x] for x in tier] == tiers


def tamper(tmp_path, name, fn_csv=None, fn_doc=None):
    art = artifacts(tmp_path, name)
    plan, csv = art / "plan.json", art / "assignment.csv"
    if fn_csv:
        csv.write_text(fn_csv(csv.read_text()))
    if fn_doc:
        doc = json.loads(plan.read_text())
        fn_doc(doc)
        plan.write_text(json.dumps(doc, indent=2))
    return run_import(plan, csv, tmp_path / "imp")


def _flip_first_rw(text):
    lines = text.splitlines(keepends=True)
    i = next(k for k, x in enumerate(lines) if x.endswith(",rw\n"))
    lines[i] = lines[i].replace(",rw\n", ",dp\n")
    return "".join(lines)


@pytest.mark.parametrize("case,kind,needle", [
    (dict(fn_csv=_flip_first_rw), "ValidationError", "the cuts say"),
    (dict(fn_csv=lambda s: s[: s.rindex("\n", 0, len(s) - 1) + 1]), "ValidationError", "total_rows"),
    (dict(fn_csv=lambda s: s.replace("table_id,row_id,tier", "table,row,tier", 1)), "ConfigError", "header"),
    (dict(fn_csv=lambda s: s.replace(",rw\n", ",xx\n", 1)), "ConfigError", "malformed line"),
    (dict(fn_doc=lambda d: d["dp_rows"][0].__setitem__(1, d["dp_rows"][0][1] + 1)), "ValidationError",
     "dp_rows differs"),
    (dict(fn_doc=lambda d: d["flex_rows"].pop()), "ValidationError", "flex_rows lists"),
    (dict(fn_doc=lambda d: d["topology"].__setitem__("a2a_intra_gibs", 1.0)), "ConfigError",
     "degenerate topology"),
])
def test_import_rejects_inconsistent_files(case, kind, needle, tmp_path):
    code, err = tamper(tmp_path, "mixed_3tier", **case)
    assert code == 3 and err.startswith(kind) and needle in err, err


def test_import_missing_files(tmp_path):
    art = artifacts(tmp_path, "zipf_2tier_1x8")
    code, err = run_import(art / "nope.json", art / "assignment.csv", tmp_path / "a")
    assert code == 3 and "plan: cannot open" in err
    code, err = run_import(art / "plan.json", art / "nope.csv", tmp_path / "b")
    assert code == 3 and "assignment: cannot open" in err


def test_keymap_config_errors_precede_device():
    import paper_2301_02959_b200 as ts
    with pytest.raises(ts.TSError) as e:
        ts.KeyMap(np.array([0, 0], np.uint32), np.array([0, 10**9], np.uint64))
    assert e.value.kind == "ConfigError" and "too sparse" in e.value.message
    with pytest.raises(ts.TSError) as e:
        ts.KeyMap(np.array([1 << 25], np.uint32), np.array([0], np.uint64))
    assert e.value.kind == "ConfigError" and "2^24" in e.value.message


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_keymap_lookup_matches_dict(cuda, tmp_path):
    import torch
    import paper_2301_02959_b200 as ts
    art = artifacts(tmp_path, "mixed_3tier")
    t, r, _ = read_assignment(art / "assignment.csv")
    km = ts.KeyMap(t, r)
    canon = {(int(a), int(b)): i for i, (a, b) in enumerate(zip(t, r))}
    rng = np.random.default_rng(3)
    pick = rng.integers(0, t.size, 50000)
    qt, qr = t[pick].copy(), r[pick].copy()
    # absent keys: unknown table, row past the table's span, row inside the span but unlisted
    qt[:3] = [7, 0, 5]
    qr[:3] = [0, 10**6, 1]
    expect = np.array([canon.get((int(a), int(b)), 0xFFFFFFFF) for a, b in zip(qt, qr)], np.uint32)
    d_t = torch.from_numpy(qt.view(np.int32)).cuda()
    d_r = torch.from_numpy(qr.view(np.int64)).cuda()
    d_c = torch.empty(qt.size, dtype=torch.int32, device="cuda")
    misses = km.lookup_device(d_t.data_ptr(), d_r.data_ptr(), qt.size, d_c.data_ptr())
    got = d_c.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, expect)
    assert misses == int((expect == 0xFFFFFFFF).sum()) >= 2
    km.close()


@pytest.mark.gpu
def test_keymap_rejects_duplicates(cuda):
    import paper_2301_02959_b200 as ts
    with pytest.raises(ts.TSError) as e:
        ts.KeyMap(np.array([0, 1, 0], np.uint32), np.array([4, 4, 4], np.uint64))
    assert e.value.kind == "ValidationError" and "duplicate" in e.value.message


@pytest.mark.gpu
@pytest.mark.parametrize("opt", [0, 1])
def test_forward_keys_equals_canonical_forward(cuda, tmp_path, opt):
    import torch
    import paper_2301_02959_b200 as ts
    art = artifacts(tmp_path, "mixed_3tier")
    code, err = run_import(art / "plan.json", art / "assignment.csv", tmp_path / "imp")
    assert code == 0, err
    s, t, r, _ = load_import(tmp_path / "imp")
    n, dim = int(s["rows"]), 32
    rng = np.random.default_rng(5)
    rows = rng.integers(0, n, 20000).astype(np.uint32)
    tabs = []
    for use_keys in (False, True):
        tab = ts.Table(n_rows=n, dim=dim, dp_cut=s["dp_cut"], flex_cut=s["flex_cut"], optimizer=opt,
                       lr=0.05, max_occurrences=rows.size, weight_seed=9)
        out = torch.empty((rows.size, dim), dtype=torch.float32, device="cuda")
        if use_keys:
            km = ts.KeyMap(t, r)
            d_t = torch.from_numpy(t[rows].view(np.int32)).cuda()
            d_r = torch.from_numpy(r[rows].view(np.int64)).cuda()
            tab.forward_keys(km, d_t.data_ptr(), d_r.data_ptr(), rows.size, out.data_ptr())
        else:
            d_rows = torch.from_numpy(rows.view(np.int32)).cuda()
            tab.forward(d_rows.data_ptr(), rows.size, out.data_ptr())
        tab.backward(out.data_ptr())
        tab.synchronize()
        wts, st = tab.read_rows(np.arange(n, dtype=np.uint32), with_state=True)
        tabs.append((out.cpu().numpy(), wts, st, tab.loss()))
        tab.close()
    (o0, w0, s0, l0), (o1, w1, s1, l1) = tabs
    assert np.array_equal(o0.view(np.uint32), o1.view(np.uint32))
    assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert np.array_equal(s0.view(np.uint32), s1.view(np.uint32))
    assert l0 == l1
    # oracle: the same update on canonical ids
    w_ref = orc.init_table(9, n, dim)
    st_ref = np.zeros(n, np.float32)
    orc.backward_update(w_ref, st_ref, rows, orc.gather(w_ref, rows), opt, 0.05, 1e-8)
    assert np.array_equal(w1.view(np.uint32), w_ref.view(np.uint32))


@pytest.mark.gpu
def test_forward_keys_two_tables_share_a_keymap(cuda, tmp_path):
    """Two tables, one key map, interleaved: forward_keys(A), forward_keys(B),
    backward(A), backward(B).  Each table's backward must see its own ids
    (the map keeps one canonical-id scratch per table)."""
    import torch
    import paper_2301_02959_b200 as ts
    art = artifacts(tmp_path, "mixed_3tier")
    code, err = run_import(art / "plan.json", art / "assignment.csv", tmp_path / "imp")
    assert code == 0, err
    s, t, r, _ = load_import(tmp_path / "imp")
    n, dim = int(s["rows"]), 32
    rng = np.random.default_rng(8)
    batches = [rng.integers(0, n, 9000).astype(np.uint32), rng.integers(0, n, 7000).astype(np.uint32)]
    km = ts.KeyMap(t, r)
    tabs, outs, keep = [], [], []
    for k, rows in enumerate(batches):
        tab = ts.Table(n_rows=n, dim=dim, dp_cut=s["dp_cut"], flex_cut=s["flex_cut"], optimizer=1, lr=0.05,
                       max_occurrences=rows.size, weight_seed=20 + k)
        out = torch.empty((rows.size, dim), dtype=torch.float32, device="cuda")
        d_t = torch.from_numpy(t[rows].view(np.int32)).cuda()
        d_r = torch.from_numpy(r[rows].view(np.int64)).cuda()
        tab.forward_keys(km, d_t.data_ptr(), d_r.data_ptr(), rows.size, out.data_ptr())
        tabs.append(tab)
        outs.append(out)
        keep += [d_t, d_r]
    for tab, out in zip(tabs, outs):
        tab.backward(out.data_ptr())
    for k, (tab, rows) in enumerate(zip(tabs, batches)):
        tab.synchronize()
        w = tab.read_rows(np.arange(n, dtype=np.uint32))
        w_ref = orc.init_table(20 + k, n, dim)
        st_ref = np.zeros(n, np.float32)
        orc.backward_update(w_ref, st_ref, rows, orc.gather(w_ref, rows), 1, 0.05, 1e-8)
        assert np.array_equal(w.view(np.uint32), w_ref.view(np.uint32)), k
        tab.close()
    km.close()


@pytest.mark.gpu
def test_forward_keys_rejects_absent_key(cuda, tmp_path):
    import torch
    import paper_2301_02959_b200 as ts
    art = artifacts(tmp_path, "zipf_2tier_1x8")
    t, r, _ = read_assignment(art / "assignment.csv")
    tab = ts.Table(n_rows=t.size, dim=32, dp_cut=0, flex_cut=0, max_occurrences=16)
    km = ts.KeyMap(t, r)
    qt = np.array([t[0], 99], np.uint32)
    qr = np.array([r[0], 0], np.uint64)
    d_t = torch.from_numpy(qt.view(np.int32)).cuda()
    d_r = torch.from_numpy(qr.view(np.int64)).cuda()
    out = torch.empty((2, 32), dtype=torch.float32, device="cuda")
    with pytest.raises(ts.TSError) as e:
        tab.forward_keys(km, d_t.data_ptr(), d_r.data_ptr(), 2, out.data_ptr())
    assert e.value.kind == "ValidationError" and "absent from the plan" in e.value.message
    tab.close()


@pytest.mark.gpu
def test_cpp_example_from_plan_files(cuda, tmp_path):
    """The C++ drop-in flow from on-disk plan files: load_device_plan ->
    KeyMap -> SequenceEmbedding(DevicePlan) -> forward_keys / backward."""
    art = artifacts(tmp_path, "mixed_3tier")
    proc = subprocess.run([str(EXAMPLE), "--plan", str(art / "plan.json"), str(art / "assignment.csv"), "3"],
                          capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    doc = json.loads(proc.stdout.strip().splitlines()[-1])
    assert doc["occurrences"] > 0 and doc["last_loss"] > 0
