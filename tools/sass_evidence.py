"""SASS evidence of the hot kernels in the in-tree libomprt_b200.so (runs
here, no GPU): per kernel, the counts of the instructions that prove the
design — UBLKCP (TMA bulk copy), SYNCS.* (mbarrier transaction counts),
LDGSTS (cp.async), LDG.E.*.256 / .128 (vector loads), SHFL, ATOMG — and the
registers / stack ptxas gave it.

    python tools/sass_evidence.py > profiles/r2_sass_evidence.json
"""

from __future__ import annotations

import collections
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2106_03219_b200" / "libomprt_b200.so"

KERNELS = (
    "k_reduce_bulk<double, 0, 3, 49152, false>",
    "k_axpy_minmax_bulk<4, 16384, 4, 256>",
    "k_dot_bulk<2, 49152, 4>",
    "k_generic<long, 0, 2, false, false, 288, 7>",
    "k_generic<double, 0, 2, false, false, 288, 7>",
    "k_generic<double, 0, 4, true, false, 288, 4>",
    "k_reduce_ext<double, 1, 3, 49152, 384>",
    "k_axpy_minmax_ext<4, 16384, 512>",
    "k_reduce_ordered_rows<double, 0, 64>",
    "k_minmax_ordered_rows<128>",
    "k_dot_ordered_rows<64>",
)
PREFIXES = ("UBLKCP", "SYNCS", "LDGSTS", "LDGDEPBAR", "LDG", "STG", "LDS", "SHFL", "ATOMG", "RED",
            "BAR", "MEMBAR", "FENCE", "UTC", "DADD", "DFMA", "FFMA", "FMNMX", "REDUX")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.split("\n")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", str(LIB)], capture_output=True,
                         text=True).stdout
    usage = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*(REG:\d+.*)", res):
        usage[m.group(1)] = dict(kv.split(":") for kv in m.group(2).split() if ":" in kv)
    parts = re.split(r"\n\s*Function : ", sass)[1:]
    names = [p.split("\n", 1)[0].strip() for p in parts]
    dem = demangle(names)
    out = {"library": str(LIB.relative_to(ROOT)), "arch": "sm_100a", "kernels": []}
    for mangled, d, body in zip(names, dem, parts):
        pick = next((k for k in KERNELS if k in d), None)
        if pick is None:
            continue
        ops = collections.Counter()
        for line in body.split("\n"):
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
            if m and m.group(1).startswith(PREFIXES):
                ops[m.group(1)] += 1
        u = usage.get(mangled, {})
        out["kernels"].append({"kernel": d.split("(")[0].replace("omprt::", ""),
                               "registers": int(u.get("REG", -1)), "stack": int(u.get("STACK", -1)),
                               "sass_counts": dict(sorted(ops.items()))})
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
