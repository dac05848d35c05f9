"""Shared test helpers (test infrastructure)."""

from __future__ import annotations

from functools import lru_cache

from oracle import oracle as O

KIND = {"add": O.A_ADD, "max": O.A_MAX, "min": O.A_MIN, "xchg": O.A_XCHG, "cas": O.A_CAS,
        "inc": O.A_INC}
DT = {"i32": O.I32, "u32": O.U32, "i64": O.I64, "u64": O.U64}
OPS = {"add": O.ADD, "max": O.MAX, "min": O.MIN}


def linearizable(kind: int, dtype: int, init: int, ops, desired, olds, final) -> bool:
    """Is there an order of the single-RMW threads whose replay through the
    oracle's step semantics yields exactly the observed old values and final
    cell?  (SPEC acceptance criterion 5; brute force with memoisation over the
    set of threads already placed.)"""
    n = len(ops)
    ops = list(ops)
    desired = list(desired) if desired is not None else [0] * n
    olds = list(olds)

    @lru_cache(maxsize=None)
    def search(done: int, cell: int) -> bool:
        # ops that observed this value and leave it unchanged (failed CAS,
        # non-raising max, xchg of the same value) can be placed right now
        # without loss of generality: they do not change what others see
        changed = True
        while changed:
            changed = False
            for g in range(n):
                if not done >> g & 1 and olds[g] == cell:
                    if O.atomic_step(kind, dtype, cell, ops[g], desired[g])[0] == cell:
                        done |= 1 << g
                        changed = True
        if done == (1 << n) - 1:
            return cell == final
        tried = set()
        for g in range(n):
            if done >> g & 1 or olds[g] != cell:
                continue
            key = (ops[g], desired[g])
            if key in tried:  # identical pending ops are interchangeable
                continue
            tried.add(key)
            new, _ = O.atomic_step(kind, dtype, cell, ops[g], desired[g])
            if search(done | (1 << g), new):
                return True
        return False

    return search(0, init)


def linearizable_programs(dtype: int, init: int, programs, olds, final) -> bool:
    """Per-thread programs of RMWs on one cell (programs[g] = [(kind, e, d)],
    olds[g] = observed old values): is there an interleaving that respects
    every thread's program order and reproduces all observations?  (SPEC
    acceptance criterion 5; DFS over per-thread program counters.)"""
    n = len(programs)
    progs = [list(p) for p in programs]
    obs = [list(o) for o in olds]

    @lru_cache(maxsize=None)
    def search(pcs: tuple, cell: int) -> bool:
        pcs = list(pcs)
        changed = True
        while changed:  # ops that observe `cell` and keep it: place now (w.l.o.g.)
            changed = False
            for g in range(n):
                k = pcs[g]
                if k < len(progs[g]) and obs[g][k] == cell:
                    kind, e, d = progs[g][k]
                    if O.atomic_step(kind, dtype, cell, e, d)[0] == cell:
                        pcs[g] += 1
                        changed = True
        if all(pcs[g] == len(progs[g]) for g in range(n)):
            return cell == final
        for g in range(n):
            k = pcs[g]
            if k < len(progs[g]) and obs[g][k] == cell:
                kind, e, d = progs[g][k]
                new, _ = O.atomic_step(kind, dtype, cell, e, d)
                nxt = list(pcs)
                nxt[g] += 1
                if search(tuple(nxt), new):
                    return True
        return False

    return search(tuple([0] * n), init)


def fold_int(op: str, bits: int, signed: bool, init: int, vals) -> int:
    """Python restatement of the integer combine (wrap / signed compare)."""
    m = (1 << bits) - 1

    def sv(v):
        v &= m
        return v - (1 << bits) if signed and v >> (bits - 1) else v

    acc = sv(init)
    for v in vals:
        v = sv(v)
        if op == "add":
            acc = sv(acc + v)
        elif op == "max":
            acc = v if acc < v else acc
        else:
            acc = v if acc > v else acc
    return acc


def uninit_script(rec) -> tuple[list, int]:
    """The vgpu check_uninit golden (gen_golden.UNINIT_SRC) as an arena script;
    returns (script, index of the READ op)."""
    script = []
    if rec["pad"]:
        script.append([0, rec["pad"], 0, 0])
    off = (rec["pad"] + 7) // 8 * 8
    v = rec["value"] - (1 << 64) if rec["value"] >> 63 else rec["value"]
    script += [[0, 64, 0, 0], [2, 8, off + 8 * rec["w"], v], [3, 8, off + 8 * rec["r"], 0],
               [1, 64, off, 0]]
    if rec["pad"]:
        script.append([1, rec["pad"], 0, 0])
    return script, 3 if rec["pad"] else 2
