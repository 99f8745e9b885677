"""Self-checking build (compute-sanitizer is closed on this pool, so the
library checks itself): _eco_b200_checked.so counts
every gather of J_{k+1} or of a tile's shared-memory band that would leave
its buffer, and every stage output element not written exactly once (the
reference's single-writer rule).  tools/sanitize_cases.py drives every
kernel family -- toys, C1, perturb_ties, wide rows, the slab emulation, both
closed-loop modes, a batch, full-size C2 and C3 stages -- on it."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2104_01284_b200" / "_eco_b200_checked.so"
pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not LIB.exists(), reason="checked build missing (run __graft_entry__.build())")
def test_checked_build_reports_no_violations():
    env = dict(os.environ, ECO_B200_LIB=str(LIB))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_cases.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert "checks bounds_violations=0 writer_violations=0" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0
