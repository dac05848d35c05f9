"""forge → B200 bridge: let the reference's own host program drive the B200
path.

forge's `HostProgram._exec_target` (host.py:501-534) calls the module-level
`tgt_target` (host.py:255-296) for every offload region and runs the
sequential fallback when it returns 1.  `install()` points that name at
`b200_tgt_target`, which

  1. recovers the region's AST from the TargetCall (the fallback closure
     carries it, host.py:366-368),
  2. recognises the `for_static_init` + per-thread fold + atomic-combine
     reduction idiom (corpus.PARTIAL_SUMS, corpus.py:219-247, and its
     max/min forms) symbolically, and
  3. runs it as one `omprt_reduce` construct launch on the GPU, with forge's
     own marshalling (_pack_arg / _write_back, host.py:209-230) and status
     contract (0 ran, 1 not runnable here → forge's fallback, 2 trap).

Regions of any other shape return 1, exactly as an unsupported device would
in the reference, and forge executes them on its host fallback.  forge is
imported lazily from the calling process; the product package never needs it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import runtime

DEVICE = "b200"
_NP = {"i32": np.int32, "u32": np.uint32, "i64": np.int64, "u64": np.uint64}
_BITS = {"i32": 32, "u32": 32, "i64": 64, "u64": 64}


@dataclass
class ReducePlan:
    """A recognised reduction region."""

    op: str            # add | max | min
    elem: str          # element type of part / cell / x
    cell: str          # captured buffer receiving the combine
    src: str | None    # captured buffer folded (None: the iteration number itself)
    lb: object         # forge Expr for the first iteration
    ub: object         # forge Expr for the last iteration
    nthreads: object   # forge Expr for the for_static_init thread count
    init: object       # forge Expr the part starts from (None: first element)


class Unrecognised(Exception):
    pass


# ------------------------------------------------------------------ matching

def _A():
    from forge import ast as A

    return A


def _name(e) -> str | None:
    A = _A()
    return e.ident if isinstance(e, A.Name) else None


def _strip_cast(e):
    A = _A()
    while isinstance(e, A.Cast):
        e = e.operand
    return e


def _is_call(e, callee: str) -> bool:
    A = _A()
    return isinstance(e, A.Call) and e.callee == callee and not e.args


def _is_flat_id(e) -> bool:
    """team_id * num_threads + thread_id (either operand order of + and *)."""
    A = _A()
    e = _strip_cast(e)
    if not (isinstance(e, A.Binary) and e.op == "+"):
        return False
    for mul, tid in ((e.left, e.right), (e.right, e.left)):
        mul, tid = _strip_cast(mul), _strip_cast(tid)
        if _is_call(tid, "omp_thread_id") and isinstance(mul, A.Binary) and mul.op == "*":
            a, b = _strip_cast(mul.left), _strip_cast(mul.right)
            if {getattr(a, "callee", None), getattr(b, "callee", None)} == \
                    {"omp_team_id", "omp_num_threads"}:
                return True
    return False


def _index_of(e, arr: str, k: int) -> bool:
    A = _A()
    return (isinstance(e, A.Index) and _name(e.base) == arr and isinstance(e.index, A.IntLit)
            and e.index.value == k)


def _fold_step(stmt, part: str, ivar: str):
    """part = part + E  |  if (part < E) { part = E; }  |  if (part > E) { part = E; }
    Returns (op, E)."""
    A = _A()
    if isinstance(stmt, A.Assign) and _name(stmt.target) == part:
        v = stmt.value
        if isinstance(v, A.Binary) and v.op == "+":
            if _name(v.left) == part:
                return "add", v.right
            if _name(v.right) == part:
                return "add", v.left
    if isinstance(stmt, A.If) and not stmt.else_body and len(stmt.then_body) == 1:
        c, body = stmt.cond, stmt.then_body[0]
        if isinstance(c, A.Binary) and c.op in ("<", ">") and _name(c.left) == part and \
                isinstance(body, A.Assign) and _name(body.target) == part and \
                body.value == c.right:
            return ("max" if c.op == "<" else "min"), c.right
    raise Unrecognised("loop body is not a fold")


def _operand(e, ivar: str):
    """E(i) = i (cast) or buf[i] (cast) -> (src buffer or None)."""
    A = _A()
    e = _strip_cast(e)
    if _name(e) == ivar:
        return None
    if isinstance(e, A.Index) and _name(_strip_cast(e.index)) == ivar and _name(e.base):
        return _name(e.base)
    raise Unrecognised("fold operand is not x[i] or i")


def _loop(stmts, part: str, bounds: str):
    """i = bounds[0]; while (i <= bounds[1]) { fold; i = i + 1; } -> (op, E, ivar)."""
    A = _A()
    if len(stmts) != 2:
        raise Unrecognised("loop shape")
    init, loop = stmts
    if not (isinstance(init, A.Assign) and _name(init.target) and _index_of(init.value, bounds, 0)):
        raise Unrecognised("loop start")
    ivar = _name(init.target)
    if not (isinstance(loop, A.While) and isinstance(loop.cond, A.Binary) and
            loop.cond.op == "<=" and _name(loop.cond.left) == ivar and
            _index_of(loop.cond.right, bounds, 1) and len(loop.body) == 2):
        raise Unrecognised("loop condition")
    step, inc = loop.body
    if not (isinstance(inc, A.Assign) and _name(inc.target) == ivar and
            isinstance(inc.value, A.Binary) and inc.value.op == "+" and
            _name(inc.value.left) == ivar and isinstance(inc.value.right, A.IntLit) and
            inc.value.right.value == 1):
        raise Unrecognised("loop increment")
    op, e = _fold_step(step, part, ivar)
    return op, e, ivar


def _combine(stmt, part: str):
    """[old =] __atomic_OP(cell, part) -> (op, cell)."""
    A = _A()
    e = stmt.value if isinstance(stmt, A.Assign) else getattr(stmt, "expr", None)
    if isinstance(stmt, A.AtomicIntrinsic):
        kind, x, v = stmt.kind.name, stmt.x, stmt.e
    elif isinstance(e, A.Call) and e.callee in ("__atomic_add", "__atomic_max", "__atomic_min") \
            and len(e.args) == 2:
        kind, x, v = e.callee[len("__atomic_"):].upper(), e.args[0], e.args[1]
        kind = {"ADD": "ATOMIC_ADD", "MAX": "ATOMIC_MAX", "MIN": "ATOMIC_MIN"}[kind]
    else:
        raise Unrecognised("no atomic combine")
    ops = {"ATOMIC_ADD": "add", "ATOMIC_MAX": "max", "ATOMIC_MIN": "min"}
    if kind not in ops or _name(v) != part or not _name(x):
        raise Unrecognised("combine shape")
    return ops[kind], _name(x)


def recognise(region) -> ReducePlan:
    """Match a forge TargetRegion against the reduction idiom."""
    A = _A()
    body = [s for s in region.body if not isinstance(s, A.LocalDecl)]
    types = {s.name: s.ty.value for s in region.body if isinstance(s, A.LocalDecl)}
    i = 0
    gname = None
    if i < len(body) and isinstance(body[i], A.Assign) and _is_flat_id(body[i].value):
        gname = _name(body[i].target)
        i += 1
    if i >= len(body) or not isinstance(body[i], A.ExprStmt) or \
            not isinstance(body[i].expr, A.Call) or body[i].expr.callee != "for_static_init":
        raise Unrecognised("no for_static_init")
    lb, ub, tid, nthr, bnd = body[i].expr.args
    tid = _strip_cast(tid)
    if not ((gname and _name(tid) == gname) or _is_flat_id(tid)):
        raise Unrecognised("for_static_init tid is not the flat thread id")
    bounds = _name(bnd)
    i += 1
    rest = body[i:]
    # form A: part = C; loop; combine
    if len(rest) == 4 and isinstance(rest[0], A.Assign) and _name(rest[0].target):
        part = _name(rest[0].target)
        op, e, ivar = _loop(rest[1:3], part, bounds)
        cop, cell = _combine(rest[3], part)
        init = rest[0].value
    # form B: if (bounds[0] <= bounds[1]) { i = bounds[0]; part = E(i); i = i + 1; loop; combine }
    elif len(rest) == 1 and isinstance(rest[0], A.If) and not rest[0].else_body:
        c = rest[0].cond
        if not (isinstance(c, A.Binary) and c.op == "<=" and _index_of(c.left, bounds, 0) and
                _index_of(c.right, bounds, 1)):
            raise Unrecognised("guard shape")
        inner = rest[0].then_body
        if len(inner) != 5:
            raise Unrecognised("guarded body shape")
        st0, st1, st2 = inner[0], inner[1], inner[2]
        ivar = _name(st0.target) if isinstance(st0, A.Assign) else None
        if not (ivar and _index_of(st0.value, bounds, 0) and isinstance(st1, A.Assign) and
                _name(st1.target)):
            raise Unrecognised("guarded start")
        part = _name(st1.target)
        first = st1.value
        if not (isinstance(st2, A.Assign) and _name(st2.target) == ivar):
            raise Unrecognised("guarded increment")
        loop = inner[3]
        if not (isinstance(loop, A.While) and len(loop.body) == 2):
            raise Unrecognised("guarded loop")
        op, e = _fold_step(loop.body[0], part, ivar)
        if _operand(first, ivar) != _operand(e, ivar):
            raise Unrecognised("first element and fold read different data")
        cop, cell = _combine(inner[4], part)
        init = None
    else:
        raise Unrecognised("region tail shape")
    if cop != op:
        raise Unrecognised("fold and combine operators differ")
    src = _operand(e, ivar)
    elem = types.get(part)
    if elem not in _NP:
        raise Unrecognised("part type")
    return ReducePlan(op, elem, cell, src, lb, ub, nthr, init)


# -------------------------------------------------------------- evaluation

def _eval(e, scalars: dict, teams: int, threads: int) -> int:
    """Evaluate a launch-time expression (literals, captured scalars, casts,
    + - * and the team/thread-count queries)."""
    A = _A()
    if isinstance(e, A.IntLit):
        return e.value
    if isinstance(e, A.Cast):
        return _eval(e.operand, scalars, teams, threads)
    if isinstance(e, A.Name) and e.ident in scalars:
        return scalars[e.ident]
    if isinstance(e, A.Call) and not e.args and e.callee in ("omp_num_teams", "omp_num_threads"):
        return teams if e.callee == "omp_num_teams" else threads
    if isinstance(e, A.Binary) and e.op in ("+", "-", "*"):
        a = _eval(e.left, scalars, teams, threads)
        b = _eval(e.right, scalars, teams, threads)
        return a + b if e.op == "+" else (a - b if e.op == "-" else a * b)
    raise Unrecognised("bound is not a launch-time constant")


def _signed(v: int, elem: str) -> int:
    bits = _BITS[elem]
    v &= (1 << bits) - 1
    return v - (1 << bits) if elem in ("i32", "i64") and v >> (bits - 1) else v


# ------------------------------------------------------------------ launch

def b200_tgt_target(call, bundle, device="vgpu", force_fail: bool = False, *, grid=None,
                    sched_seed: int = 0, check_uninit: bool = False,
                    collect_trace: bool = False, out: dict | None = None) -> int:
    """forge.host.tgt_target for device "b200" (other devices go to forge's own)."""
    from forge import host as H

    arch = str(getattr(device, "arch", device))
    if arch != DEVICE:
        return _original(call, bundle, device, force_fail, grid=grid, sched_seed=sched_seed,
                         check_uninit=check_uninit, collect_trace=collect_trace, out=out)
    if call.values is None:
        raise ValueError("TargetCall is not bound to argument values")
    if force_fail or not torch.cuda.is_available():
        return 1
    region = _region_of(call)
    if region is None:
        return 1
    try:
        plan = recognise(region)
    except Unrecognised:
        return 1
    teams, threads = grid if grid is not None else (call.grid[0] or 1, call.grid[1] or 1)
    descs = {d.name: d for d in call.args}
    vals = dict(zip((d.name for d in call.args), call.values))
    scalars = {n: _signed(int(v), descs[n].elem.value) for n, v in vals.items()
               if descs[n].kind == "scalar"}
    try:
        lb = _eval(plan.lb, scalars, teams, threads)
        ub = _eval(plan.ub, scalars, teams, threads)
        n = _eval(plan.nthreads, scalars, teams, threads)
        init = None if plan.init is None else _eval(plan.init, scalars, teams, threads)
    except Unrecognised:
        return 1
    # the device schedule partitions over every launched thread; a region
    # that names another thread count is a different partition
    if n != teams * threads or plan.cell not in descs or descs[plan.cell].elem.value != plan.elem:
        return 1
    if plan.op == "add" and init not in (None, 0):
        return 1
    dt = _NP[plan.elem]
    dev = torch.device("cuda", torch.cuda.current_device())
    cell_raw = bytearray(H._pack_arg(descs[plan.cell], vals[plan.cell]))
    cell = torch.from_numpy(np.frombuffer(cell_raw, dtype=dt).copy()).to(dev)
    if plan.src is None:
        if ub >= lb and (lb < 0 or ub > (1 << 40)):
            return 1
        m = (1 << _BITS[plan.elem]) - 1
        it = np.arange(0, max(ub + 1, 1), dtype=np.int64) & m
        x = torch.from_numpy(it.astype(np.uint64).astype(dt)).to(dev)
    else:
        if plan.src not in descs or descs[plan.src].elem.value != plan.elem:
            return 1
        raw = H._pack_arg(descs[plan.src], vals[plan.src])
        x = torch.from_numpy(np.frombuffer(raw, dtype=dt).copy()).to(dev)
        if ub >= lb and (lb < 0 or ub >= x.numel()):
            if out is not None:
                out["trap"] = ("OutOfBounds", f"iteration space [{lb}, {ub}] escapes "
                               f"{plan.src}[0:{x.numel()}]")
            return 2
    out_dev = cell[:1]
    if init is not None and plan.op != "add":
        # an idempotent combine of the per-thread start value (max/min)
        out_dev.copy_(torch.from_numpy(np.array(
            [runtime_fold(plan.op, int(out_dev.cpu().item()), init, plan.elem)], dtype=dt)))
    runtime.reduce(x, plan.op, lb=lb, ub=ub, sched="static", teams=teams, threads=threads,
                   out=out_dev)
    torch.cuda.synchronize(dev)
    if out is not None:
        out["result"] = None
    H._write_back(vals[plan.cell], cell.cpu().numpy().tobytes())
    return 0


def runtime_fold(op: str, a: int, b: int, elem: str) -> int:
    a, b = _signed(a, elem), _signed(b, elem)
    return max(a, b) if op == "max" else min(a, b)


def _region_of(call):
    fb = getattr(call, "fallback", None)
    for d in getattr(fb, "__defaults__", None) or ():
        if type(d).__name__ == "TargetRegion":
            return d
    return None


_original = None


def install() -> None:
    """Route forge's offloads for device "b200" through the B200 path."""
    global _original
    from forge import host as H

    if _original is None:
        _original = H.tgt_target
    H.tgt_target = b200_tgt_target


def uninstall() -> None:
    from forge import host as H

    if _original is not None:
        H.tgt_target = _original
