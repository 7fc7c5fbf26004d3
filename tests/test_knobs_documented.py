"""Every TIERSHARD_* environment knob the native code reads is listed in
DESIGN.md's schedule-knob table (CPU only: a source scan)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_every_env_knob_is_documented():
    src = ROOT / "paper_2301_02959_b200" / "csrc"
    knobs = set()
    for f in list(src.rglob("*.cu")) + list(src.rglob("*.cpp")) + list(src.rglob("*.cuh")) + list(src.rglob("*.hpp")):
        knobs |= set(re.findall(r'getenv\("(TIERSHARD_[A-Z0-9_]+)"', f.read_text()))
    assert knobs, "no knobs found: the scan is broken"
    design = (ROOT / "DESIGN.md").read_text()
    missing = sorted(k for k in knobs if f"`{k}`" not in design)
    assert not missing, f"undocumented knobs: {missing}"
