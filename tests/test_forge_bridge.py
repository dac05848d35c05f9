"""forge drives the B200 path.

The reference package is imported from baseline/_ref (the unmodified
reference, pip-installed with --no-deps; it travels to the GPU box) or, in the
build container, from /root/reference.  The CPU tests check the region
recogniser on forge's own ASTs; the GPU tests run forge programs with
forge.host.tgt_target routed to the B200 (paper_2106_03219_b200.forge_bridge).
"""

from __future__ import annotations

import copy
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "forge" / "__init__.py").exists():
        sys.path.insert(0, str(cand))
        break
forge = pytest.importorskip("forge")

from forge import corpus  # noqa: E402
from forge.host import HostProgram, run_source  # noqa: E402
from forge.parser import parse_module  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2106_03219_b200 import forge_bridge as B  # noqa: E402

RECOGNISED = {"partial_sums"}

REDUCE_SRC = """\
void kernel({T} *x, {T} *cell, i64 n) {{
  #pragma omp target
  {{
    i64 bounds[2];
    i64 i;
    i64 g;
    {T} part;
    {T} old;
    g = (i64) (omp_team_id() * omp_num_threads() + omp_thread_id());
    for_static_init(0, n - 1, g, (i64) (omp_num_teams() * omp_num_threads()), bounds);
    if (bounds[0] <= bounds[1]) {{
      i = bounds[0];
      part = x[i];
      i = i + 1;
      while (i <= bounds[1]) {{
        {BODY}
        i = i + 1;
      }}
      old = {ATOMIC}(cell, part);
    }}
  }}
}}
"""
BODIES = {"add": ("part = part + x[i];", "__atomic_add"),
          "max": ("if (part < x[i]) { part = x[i]; }", "__atomic_max"),
          "min": ("if (part > x[i]) { part = x[i]; }", "__atomic_min")}


def region_of(src):
    prog = HostProgram(parse_module(src))
    return prog, prog.target_calls[0]


def test_recogniser_on_corpus():
    for name, src in corpus.CORPUS:
        prog, call = region_of(src)
        region = B._region_of(call)
        assert region is not None
        try:
            plan = B.recognise(region)
            ok = True
        except B.Unrecognised:
            ok = False
        assert ok == (name in RECOGNISED), name
        if ok:
            assert (plan.op, plan.elem, plan.cell, plan.src) == ("add", "u32", "cell", None)


@pytest.mark.parametrize("ty", ["i32", "u32", "i64", "u64"])
@pytest.mark.parametrize("op", ["add", "max", "min"])
def test_recogniser_on_reduction_kernels(ty, op):
    body, atomic = BODIES[op]
    prog, call = region_of(REDUCE_SRC.format(T=ty, BODY=body, ATOMIC=atomic))
    plan = B.recognise(B._region_of(call))
    assert (plan.op, plan.elem, plan.cell, plan.src, plan.init) == (op, ty, "cell", "x", None)


def test_recogniser_rejects_other_partitions():
    # a thread count that is not the launched one, a mismatched combine
    src = corpus.PARTIAL_SUMS.replace("__atomic_add(cell, part)", "__atomic_max(cell, part)")
    with pytest.raises(B.Unrecognised):
        B.recognise(B._region_of(region_of(src)[1]))


@pytest.mark.gpu
def test_forge_corpus_runs_on_b200(cuda):
    B.install()
    try:
        for name, src in corpus.CORPUS:
            want = run_source(src, device="vgpu", sched_seed=3)
            got = run_source(src, device="b200")
            assert got.stdout == want.stdout, name
            assert got.exit_status == want.exit_status == 0
            # recognised reductions run as the omprt_reduce construct, every
            # other region as its compiled sm_100a image: nothing falls back
            statuses = {s for _, s in got.offloads}
            assert statuses == {0}, (name, got.offloads)
    finally:
        B.uninstall()


@pytest.mark.gpu
def test_forge_reduction_regions_on_b200(cuda, fallback_golden):
    from forge.host import tgt_target as forge_tgt_target  # noqa: F401

    B.install()
    try:
        import forge.host as H

        for r in fallback_golden["reductions"]:
            body, atomic = BODIES[r["op"]]
            prog, call = region_of(REDUCE_SRC.format(T=r["dtype"], BODY=body, ATOMIC=atomic))
            dt = {"i32": O.I32, "u32": O.U32, "i64": O.I64, "u64": O.U64}[r["dtype"]]
            x = bytearray(O.fill(r["n"], dt, r["seed"], r["k"]).tobytes())
            cell = bytearray(np.array([r["init"]], dtype=O.NP_DTYPE[dt]).tobytes())
            vals = [{"x": x, "cell": cell, "n": r["n"]}[a.name] for a in call.args]
            st = H.tgt_target(call.bind(vals), {}, "b200", grid=(r["teams"], r["threads"]))
            assert st == 0
            got = np.frombuffer(bytes(cell), dtype=O.NP_DTYPE[dt])[0]
            assert int(got) == r["fallback"], r
    finally:
        B.uninstall()


@pytest.mark.gpu
def test_forge_collect_trace_on_b200(cuda):
    # forge's own run_source(collect_trace=True) on device "b200": the
    # recognised reduction region returns the per-team hardware trace in the
    # vgpu's line format ("seq team thread kind detail")
    B.install()
    try:
        src = dict(corpus.CORPUS)["partial_sums"]
        res = run_source(src, device="b200", collect_trace=True)
        assert res.exit_status == 0
        kinds = [ln.split()[3] for ln in res.device_traces]
        assert "atomic.inc" in kinds and kinds[-1] == "combine"
    finally:
        B.uninstall()
