"""A short run of tools/ordered_fuzz.py inside the GPU suite: random
geometries/schedules/sizes through every ORDERED path (bit-identical to the
reference order) and the SPMD paths (integers bit-exact, fp64 within 1e-6)."""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_random_launches_match_the_oracle(cuda):
    res = subprocess.run([sys.executable, str(ROOT / "tools" / "ordered_fuzz.py"), "--cases", "90",
                          "--seed", "31"], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert '"failures": 0' in res.stdout
