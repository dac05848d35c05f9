"""The C ABI from a plain C program (no Python, no torch): build here, run on
the GPU (tests/c/abi_example.c)."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2106_03219_b200"


def build_example(tmp: Path) -> Path:
    exe = tmp / "abi_example"
    cmd = ["/usr/bin/gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
           str(ROOT / "tests" / "c" / "abi_example.c"), "-L", str(PKG), "-l:libomprt_b200.so",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{PKG}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_links(tmp_path):
    assert build_example(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs_on_b200(cuda, tmp_path):
    exe = build_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"fp64 sum ([0-9.eE+-]+)", r.stdout)
    exact = O.exact_sum_gen(0, (1 << 24) - 1, O.F64)
    assert abs(float(m.group(1)) - exact) <= 1e-6 * exact
    assert "partial_sums 5050" in r.stdout and "trap kind 1 code 1" in r.stdout
