"""CPU tests of bench.py's host-side logic (no GPU): the NUMA cpulist parser,
the ncu-capture provenance check that keeps a stale capture off the bench
line, and the JSON contract's argument defaults."""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_parse_cpulist():
    assert bench.parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert bench.parse_cpulist("5") == {5}
    assert bench.parse_cpulist("\n") == set()


def _capture(tmp_path, kernel, grid=148, block=384, sha="x"):
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "ncu_bench_kernel.json").write_text(json.dumps({
        "captured_at": "2026-01-01T00:00:00Z", "src_sha16": sha,
        "dram_bytes_per_launch": 8.6e9,
        "launches": [{"kernel": kernel, "launch__grid_size": grid, "launch__block_size": block,
                      "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": 90.0}]}))


def test_ncu_capture_current(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    monkeypatch.setattr(bench, "src_sha16", lambda: "abc")
    _capture(tmp_path, f"void {bench.BENCH_KERNEL}, 0>(const T1 *)", sha="abc")
    c = bench.ncu_capture(148, 384, 1)
    assert c["traffic"] == 8.6e9 and c["frac_ncu_dram"] == 0.9
    assert c["status"].startswith("current")


@pytest.mark.parametrize("kernel,grid", [("void k_reduce_bulk<double, 0, 9, 1024, 0>()", 148),
                                         (f"void {bench.BENCH_KERNEL}>()", 296)])
def test_ncu_capture_stale_is_dropped(tmp_path, monkeypatch, kernel, grid):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    _capture(tmp_path, kernel, grid=grid)
    c = bench.ncu_capture(148, 384, 1)
    assert c["traffic"] is None and c["frac_ncu_dram"] is None
    assert c["status"].startswith("stale")


def test_ncu_capture_missing(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    assert bench.ncu_capture(148, 384, 1)["status"] == "missing"


def test_defaults_are_the_headline_config(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.gpus == 1 and a.impl == "ours" and a.warmup >= 3
    assert a.n == 1 << 30 and a.c5_n == 1 << 33 and a.sched == "distribute"


def test_committed_capture_is_of_the_bench_kernel():
    d = json.loads((ROOT / "profiles" / "ncu_bench_kernel.json").read_text())
    assert bench.BENCH_KERNEL in d["launches"][0]["kernel"]


def test_spawned_argv_survives_torchrun_parsing(monkeypatch):
    """--gpus N > 1 re-launches under torch.distributed.run; none of the
    script's options may be taken as an abbreviation of torchrun's own
    (`--n` would match --nnodes / --nproc-per-node)."""
    import subprocess

    from torch.distributed import run as trun

    captured = {}
    monkeypatch.setattr(subprocess, "call", lambda cmd: captured.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--n", "1024", "--steps", "3",
                                      "--warmup", "3", "--backend", "gloo", "--no-legs",
                                      "--teams", "4", "--threads", "64", "--exchange", "p2p"])
    bench.spawn_ranks(bench.parse())
    cmd = captured["cmd"]
    i = cmd.index("torch.distributed.run")
    ns = trun.get_args_parser().parse_args(cmd[i + 1:])
    assert ns.nproc_per_node == "8" and ns.training_script.endswith("bench.py")
    monkeypatch.setattr(sys, "argv", ["bench.py", *ns.training_script_args])
    a = bench.parse()
    assert (a.gpus, a.n, a.steps, a.backend, a.teams, a.threads, a.exchange) == \
        (8, 1024, 3, "gloo", 4, 64, "p2p")


def test_both_arms_print_the_same_config():
    """The reference arm and ours describe the workload with the same dict
    (the driver matches them); measured values stay out of `config`."""
    import inspect

    c1 = bench.workload_config(1 << 30, 1, "distribute", 148, 384)
    c8 = bench.workload_config(1 << 30, 8, "distribute", 148, 384)
    assert c1["n_global"] == 1 << 30 and c8["n_global"] == 8 << 30 and c8["parallelism"] == "dp8"
    assert not any(isinstance(v, float) for v in c1.values())
    src_ref = inspect.getsource(bench.run_reference_arm)
    src_ours = inspect.getsource(bench.run_ours)
    assert '"config": workload_config(' in src_ref and '"config": workload_config(' in src_ours
