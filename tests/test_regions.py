"""Region compiler (forge IR image -> sm_100a B200 image), CPU side.

No GPU needed: the reference's own codegen produces the nvptx64 IR image of
every golden program (tests/golden/region_programs.json, made by
oracle/gen_region_golden.py from the reference), regionc translates it and
NVRTC compiles it for sm_100a; the image container and the OMPBNDL1 bundle
with a "b200" entry round-trip through forge's own bundler.
"""

from __future__ import annotations

import json
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "forge" / "__init__.py").exists():
        sys.path.insert(0, str(cand))
        break
forge = pytest.importorskip("forge")

from forge.bundler import Bundle  # noqa: E402

from paper_2106_03219_b200 import forge_bridge as B  # noqa: E402
from paper_2106_03219_b200 import regionc as R  # noqa: E402

GOLDEN = json.loads((ROOT / "tests" / "golden" / "region_programs.json").read_text())
PROGRAMS = {p["name"]: p for p in GOLDEN["programs"]}


def nvptx_ir(src: str) -> str:
    import copy

    from forge.codegen import compile_device_image
    from forge.lowering import lower_atomics
    from forge.parser import parse_module

    return compile_device_image(lower_atomics(copy.deepcopy(parse_module(src))),
                                "nvptx64").render()


def test_ir_parser_round_trips_the_reference_ir():
    from forge.ir import parse_ir

    for p in GOLDEN["programs"]:
        text = nvptx_ir(p["source"])
        ours = R.parse_ir(text)
        ref = parse_ir(text)
        assert [f.name for f in ours.funcs] == [f.name for f in ref.funcs]
        assert [(g.name, g.space, g.ty, g.count, g.init) for g in ours.globals] == \
            [(g.name, g.space, g.ty, g.count, g.init) for g in ref.globals]
        for fo, fr in zip(ours.funcs, ref.funcs):
            assert fo.params == fr.params and fo.ret == fr.ret
            assert [(b.label, [(i.op, i.dst, i.args) for i in b.instrs]) for b in fo.blocks] == \
                [(b.label, [(i.op, i.dst, i.args) for i in b.instrs]) for b in fr.blocks]


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_every_golden_program_compiles_for_sm100a(name):
    img = R.compile_image(nvptx_ir(PROGRAMS[name]["source"]))
    assert img.cubin[:4] == b"\x7fELF"
    assert img.manifest["arch"] == "sm_100a"
    assert "__omp_offload_0" in img.kernels
    back = R.B200Image.from_bytes(img.to_bytes())
    assert back.cubin == img.cubin and back.manifest == img.manifest


def test_layout_is_the_vgpu_layout():
    img = R.compile_image(nvptx_ir(PROGRAMS["team_shared"]["source"]))
    lay = {g["name"]: (g["space"], g["off"], g["bytes"]) for g in img.manifest["globals"]}
    # vgpu._layout: 8-aligned offsets in declaration order per space (vgpu.py:171-196)
    assert lay["base"] == ("team_shared", 0, 8)
    assert lay["counter"] == ("team_shared", 8, 8)
    assert lay["scratch"] == ("team_shared", 16, 32)
    assert lay["zeros"] == ("team_shared", 48, 24)
    assert img.manifest["shared_bytes"] == 72 and img.manifest["has_barrier"]
    img = R.compile_image(nvptx_ir(PROGRAMS["global_device_data"]["source"]))
    lay = {g["name"]: (g["space"], g["off"], g["bytes"]) for g in img.manifest["globals"]}
    assert lay["table"] == ("global", 0, 16) and lay["seed"] == ("global", 16, 4)
    assert img.manifest["global_bytes"] == 20


def test_translation_rejects_foreign_targets_and_opcodes():
    text = nvptx_ir(PROGRAMS["corpus_counter_add"]["source"])
    with pytest.raises(R.RegionCompileError):
        R.translate(text.replace("target nvptx64", "target amdgcn"))
    with pytest.raises(R.RegionCompileError):
        R.translate(text.replace("add.u32", "frobnicate.u32", 1))


def test_vgpu_images_translate_too():
    from forge.codegen import compile_device_image
    from forge.lowering import lower_atomics
    from forge.parser import parse_module
    import copy

    mod = lower_atomics(copy.deepcopy(parse_module(PROGRAMS["barrier_ok"]["source"])))
    img = R.compile_image(compile_device_image(mod, "vgpu").render())
    assert img.manifest["source_target"] == "vgpu" and img.manifest["has_barrier"]


def test_bad_images_are_rejected():
    img = R.compile_image(nvptx_ir(PROGRAMS["corpus_inc_ring"]["source"])).to_bytes()
    with pytest.raises(R.BadImage):
        R.B200Image.from_bytes(b"NOTANIMG" + img[8:])
    with pytest.raises(R.BadImage):
        R.B200Image.from_bytes(img[:-1])


def test_bundle_carries_a_b200_entry():
    src = PROGRAMS["corpus_partial_sums"]["source"]
    data = B.compile_bundle(src)
    b = Bundle.from_bytes(data)
    names = [n for n, _ in b.entries]
    assert names == ["host", "vgpu", "nvptx64", "b200"]
    img = R.B200Image.from_bytes(dict(b.images)["b200"])
    assert img.manifest["ir_sha256"] == R.compile_image(nvptx_ir(src)).manifest["ir_sha256"]
    # forge's own unbundle accepts it and its vgpu run is unaffected
    res = forge.host.run_bundle(data)
    assert res.exit_status == 0 and res.stdout == PROGRAMS["corpus_partial_sums"]["stdout"]


def test_cli_compile_and_inspect(tmp_path, capsys):
    src = tmp_path / "prog.mc"
    src.write_text(PROGRAMS["corpus_counter_add"]["source"])
    assert B.main(["compile", str(src)]) == 0
    out = tmp_path / "prog.o"
    assert out.exists()
    assert B.main(["inspect", str(out)]) == 0
    text = capsys.readouterr().out
    assert "b200" in text and "sm_100a" in text and "__omp_offload_0" in text


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not on PATH")
def test_sass_uses_the_hardware_primitives(tmp_path):
    """The translation lands on the NVIDIA primitives selectors.py:84-93 names:
    BAR.RED for the team barrier, ATOM/ATOMG for the atomics, MEMBAR for fences."""
    img = R.compile_image(nvptx_ir(PROGRAMS["team_shared"]["source"]))
    f = tmp_path / "k.cubin"
    f.write_bytes(img.cubin)
    sass = subprocess.run(["cuobjdump", "-sass", str(f)], capture_output=True, text=True).stdout
    assert "BAR.RED.OR" in sass
    assert "ATOM" in sass
    assert "MEMBAR" in sass or "FENCE" in sass
