"""Per-team device trace (runtime.Trace / omprt_set_trace): the B200 analog
of the vgpu's collect_trace (vgpu.py:351-353) — one record per CTA with its
SM, its start time and the ticket its last-team-finishes atom.inc returned,
plus the ordered combine; ORDERED launches record streaming warps and the
folder.  tgt_target(collect_trace=True) renders the vgpu's line format."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import offload, runtime

pytestmark = pytest.mark.gpu


def test_team_records_and_ticket_permutation(cuda):
    x = runtime.synthetic(1 << 22, "f64", O.SEED, device=cuda)
    T = runtime.num_sms()  # one CTA per team (no split at >= SMs/2 teams)
    with runtime.Trace(cuda) as tr:
        runtime.reduce(x, sched="distribute", teams=T, threads=256)
    r = tr.records
    teams = r[r["kind"] == 1]
    comb = r[r["kind"] == 2]
    assert len(teams) == T and len(comb) == 1
    assert sorted(teams["ticket"].tolist()) == list(range(T))  # every ticket value once
    assert sorted(teams["cta"].tolist()) == list(range(T))
    assert (teams["t_end"] >= teams["t_begin"]).all()
    assert (teams["smid"] < runtime.num_sms()).all()
    # the team holding the last ticket ran the combine after every ticket was taken
    last = teams[teams["ticket"] == T - 1][0]
    assert comb[0]["cta"] == last["cta"]
    assert comb[0]["t_end"] >= teams["t_end"].max()
    lines = tr.lines()
    assert len(lines) == T + 1 and lines[-1].split()[3] == "combine"
    assert all(len(ln.split()) >= 5 for ln in lines)


def test_split_team_records_every_cta(cuda):
    x = runtime.synthetic(1 << 20, "i64", O.SEED, device=cuda)
    with runtime.Trace(cuda) as tr:
        runtime.reduce(x, teams=1, threads=128)
    teams = tr.records[tr.records["kind"] == 1]
    assert len(teams) > 1  # one OpenMP team split over several CTAs
    assert sorted(teams["ticket"].tolist()) == list(range(len(teams)))


def test_ordered_records_streams_and_folder(cuda):
    x = runtime.synthetic(1 << 22, "f64", O.SEED, device=cuda)
    with runtime.Trace(cuda) as tr:
        runtime.reduce(x, sched="distribute", teams=16, threads=256, mode="ordered")
    r = tr.records
    streams, fold = r[r["kind"] == 3], r[r["kind"] == 4]
    assert len(fold) == 1 and len(streams) >= 1
    assert int(streams["ticket"].sum()) == (16 * 256 + 31) // 32  # every group folded once
    assert fold[0]["t_end"] >= streams["t_end"].max()


def test_no_records_without_a_trace(cuda):
    x = runtime.synthetic(1 << 16, "f64", O.SEED, device=cuda)
    tr = runtime.Trace(cuda)
    runtime.reduce(x, teams=8, threads=128)
    torch.cuda.synchronize()
    assert int(tr.buf.abs().sum().item()) == 0


def test_tgt_target_collect_trace(cuda):
    n = 100_000
    x = O.fill(n, O.I64, O.SEED, 1)
    call = offload.TargetCall(0, offload.kernel_name(0),
                              (offload.ArgDescriptor("n", "scalar", "i64"),
                               offload.ArgDescriptor("x", "buffer", "i64"),
                               offload.ArgDescriptor("cell", "buffer", "i64")), grid=(4, 64))
    cell = bytearray(8)
    image = {"b200": {offload.kernel_name(0): offload.RegionKernel(
        "reduce", {"x": "x", "cell": "cell", "n": "n"}, op="add")}}
    out: dict = {}
    st = offload.tgt_target(call.bind([n, x.tobytes(), cell]), image, "b200",
                            collect_trace=True, out=out)
    assert st == 0
    assert int(np.frombuffer(bytes(cell), dtype=np.int64)[0]) == int(x.sum())
    kinds = [ln.split()[3] for ln in out["trace"]]
    assert kinds.count("atomic.inc") >= 4 and kinds[-1] == "combine"


def test_generic_mode_records_while_traced(cuda):
    # generic mode launches its traced instance only while a ring is installed
    x = runtime.synthetic(1 << 20, "i64", O.SEED, device=cuda)
    with runtime.Trace(cuda) as tr:
        runtime.generic_reduce(x, teams=64, par_threads=128)
    teams = tr.records[tr.records["kind"] == 1]
    assert len(teams) == 64 and sorted(teams["ticket"].tolist()) == list(range(64))
    assert len(tr.records[tr.records["kind"] == 2]) == 1
    after = runtime.Trace(cuda)
    runtime.generic_reduce(x, teams=64, par_threads=128)
    torch.cuda.synchronize()
    assert int(after.buf.abs().sum().item()) == 0
