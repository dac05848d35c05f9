"""INTEGRATION.md stays in step with the code: every Python snippet parses,
and every omprt_* entry point the document names is declared in
include/omprt_b200.h and exported by the library (CPU only)."""

import ast
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
DOC = (ROOT / "INTEGRATION.md").read_text()
HEADER = (ROOT / "include" / "omprt_b200.h").read_text()


def test_python_snippets_parse():
    blocks = re.findall(r"```python\n(.*?)```", DOC, flags=re.S)
    assert blocks
    for b in blocks:
        ast.parse(b)


def test_named_entry_points_exist():
    from paper_2106_03219_b200 import _lib

    names = set(re.findall(r"\bomprt_[a-z0-9_]+(?=\s*\()", DOC))
    assert names
    declared = set(re.findall(r"\b(omprt_[a-z0-9_]+)\s*\(", HEADER))
    missing = sorted(n for n in names if n not in declared)
    assert not missing, missing
    lib = _lib.load(build_if_missing=True)
    for n in names:
        assert hasattr(lib, n), n
