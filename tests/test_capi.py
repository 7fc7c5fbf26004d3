"""The drop-in boundary: libtiershard_b200.so loads, exports every entry point
include/tiershard_b200.h declares, and fails loudly (no CPU fallback) where
no device is present."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2301_02959_b200 as ts
from paper_2301_02959_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "tiershard_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ts_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(capi.EXPORTS) == declared_symbols()


def test_library_exports_every_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(capi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ts.load()
    for s in declared_symbols():
        assert hasattr(lib, s)
    assert lib.ts_abi_version() == 2
    assert "sm_100a" in ts.build_info()


def test_no_cpu_fallback_without_device():
    if ts.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(ts.TSError) as e:
        ts.Table(n_rows=10, dim=32, dp_cut=0, flex_cut=0)
    assert e.value.kind == "NoDevice"
    with pytest.raises(ts.TSError) as e:
        ts.Router(10, 0, 0, np.zeros(10, np.uint8), 1, 1)
    assert e.value.kind == "NoDevice"
    assert "no CPU fallback" in e.value.message


def test_group_host_side():
    """ts_group is host-only until a table attaches: create / destroy work
    without a device, bad sizes are ConfigErrors."""
    g = ts.Group(4)
    assert g.ranks == 4 and g.handle
    g.close()
    for bad in (0, 257):
        with pytest.raises(ts.TSError) as e:
            ts.Group(bad)
        assert e.value.kind == "ConfigError"


def test_keymap_rejects_huge_row_ids_before_device():
    """row_id + 1 must not wrap the dense map's span: rejected on
    the host, before any device work."""
    with pytest.raises(ts.TSError) as e:
        ts.KeyMap(np.array([0, 0], np.uint32), np.array([5, 2**64 - 1], np.uint64))
    assert e.value.kind == "ConfigError" and "too large" in e.value.message


def test_config_errors_before_device():
    with pytest.raises(ts.TSError) as e:
        ts.Router(10, 5, 2, np.zeros(10, np.uint8), 1, 1)
    assert e.value.kind == "ValidationError"
    assert "plan does not cover" in e.value.message


EXAMPLE = ROOT / "paper_2301_02959_b200" / "bin" / "ts_example"


def test_cpp_example_fails_loudly_without_device():
    """The C++ front door (tiershard/device.hpp) plans on the host, then
    refuses to run the table anywhere but a GPU."""
    if ts.device_count() > 0:
        pytest.skip("a device is present")
    proc = subprocess.run([str(EXAMPLE), "20000", "32", "64", "1"], capture_output=True, text=True,
                          timeout=300)
    assert proc.returncode == 3
    assert "no CUDA device" in proc.stdout


@pytest.mark.gpu
def test_cpp_example_trains_on_device(cuda):
    import json
    proc = subprocess.run([str(EXAMPLE), "100000", "64", "128", "3"], capture_output=True, text=True,
                          timeout=300)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    doc = json.loads(proc.stdout.strip().splitlines()[-1])
    assert doc["occurrences"] > 0 and doc["served"] > 0
    assert doc["last_loss"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("nodes,w", [(1, 2), (2, 2)])
def test_cpp_example_in_process_group(cuda, nodes, w):
    """The C++ front door with a DeviceGroup: U ranks as threads of one
    process (tiershard::DeviceGroup, DeviceOptions::group), every rank
    stepping its slice of the reference Workload through train_steps_host;
    the summed SERVED counters equal the last iteration's occurrences."""
    import json
    proc = subprocess.run([str(EXAMPLE), "--group", str(nodes), str(w), "50000", "3"], capture_output=True,
                          text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    doc = json.loads(proc.stdout.strip().splitlines()[-1])
    assert doc["ranks"] == nodes * w
    assert doc["served"] == doc["last_iteration_occurrences"] > 0
    assert doc["last_loss_sum"] > 0
