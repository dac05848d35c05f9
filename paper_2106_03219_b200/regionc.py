"""Region compiler: forge device images (IR) -> sm_100a cubins ("B200 images").

The reference compiles every offload region into a per-target IR image
(codegen.compile_device_image, codegen.py:555-561) and bundles those images
next to the host program (bundler.py:37-98).  Only the `vgpu` image can run
— on a Python interpreter (vgpu.py); the `nvptx64` image is IR only
(host.py:62, 270).  This module is the missing device backend:
it translates an IR image (the `nvptx64` one, whose intrinsic table names
exactly the primitives of selectors.py:84-93, or the `vgpu` one) into CUDA
C++ over the runtime in csrc/region_rt.cuh and compiles it with NVRTC for
sm_100a.  The result is a `B200Image`: a cubin plus a JSON manifest (kernel
parameter lists, the vgpu memory layout of globals and team-shared data, and
the trap-site table that turns a device trap record into the vgpu's message).

Semantics follow the vgpu instruction by instruction (vgpu.py:384-625):
wrapping fixed-width integer ALU, truncating signed division with
DivideByZero, bounds-checked fat pointers (OutOfBounds), 0xAA poison for
slots and loader_uninitialized data, check_uninit shadow, seq_cst atomics,
team barriers that trap Deadlock when they meet a finished thread.  What the
vgpu's seeded interleaving decides (the order of racing atomics) is decided by
the hardware here; interleaving-independent programs (corpus.CORPUS) produce
identical results.

The IR text format is parsed here (a restatement of ir.parse_ir, ir.py:143-233),
so loading and running B200 images needs neither forge nor NVRTC; compiling
needs NVRTC (libnvrtc, shipped with CUDA 12.9 in this image).
"""

from __future__ import annotations

import ctypes
import ctypes.util
import hashlib
import json
import os
import re
import struct
from dataclasses import dataclass, field
from pathlib import Path

CSRC = Path(__file__).resolve().parent / "csrc"
IMAGE_MAGIC = b"OMPB200\x01"
ARCH = "sm_100a"
KERNEL_PREFIX = "__omp_offload_"          # codegen.py:59-63
GLOBAL_ALIGN = 8                          # vgpu.py:20
SHARED_CAPACITY = 131072                  # vgpu.py:22, selectors.py:60
_SIZES = {"i32": 4, "u32": 4, "i64": 8, "u64": 8}
_SIGNED = {"i32", "i64"}
ARGV_HEADER = 5                           # trap, globals, gshadow, sshadow, waitmask


class RegionCompileError(Exception):
    """The image cannot be translated or NVRTC rejected the translation."""


class BadImage(Exception):
    """Bytes that are not a B200 image (wrong magic, truncated, bad manifest)."""


# ------------------------------------------------------------------ IR model
# (ir.py:22-120, restated: the product must not import the reference)

@dataclass
class Global:
    name: str
    space: str
    ty: str
    count: int
    init: object


@dataclass
class Slot:
    name: str
    ty: str
    count: int | None


@dataclass
class Ins:
    op: str
    dst: str | None
    args: list[str]


@dataclass
class Block:
    label: str
    instrs: list[Ins] = field(default_factory=list)


@dataclass
class Func:
    name: str
    params: list[tuple[str, str]]
    ret: str | None
    slots: list[Slot] = field(default_factory=list)
    blocks: list[Block] = field(default_factory=list)


@dataclass
class Module:
    target: str
    globals: list[Global] = field(default_factory=list)
    funcs: list[Func] = field(default_factory=list)


_GLOBAL_RE = re.compile(r"^global @([\w.]+) space=(global|team_shared) type=(\w+) "
                        r"count=(\d+) init=(zero|none|-?\d+)$")
_FUNC_RE = re.compile(r"^func @([\w.]+)\((.*)\) -> (\w+(?:<\w+>)?|void) \{$")
_PARAM_RE = re.compile(r"^%([\w.]+): (\w+(?:<\w+>)?)$")
_SLOT_RE = re.compile(r"^  local %([\w.]+): (?:\[(\d+) x (\w+)\]|(\w+))$")
_LABEL_RE = re.compile(r"^(bb\d+):$")
_INSTR_RE = re.compile(r"^  (?:%([\w.]+) = )?([\w.]+)(?: (.*))?$")
_CALL_RE = re.compile(r"^(@[\w.]+)\((.*)\)$")


def parse_ir(text: str) -> Module:
    """Parse the reference's textual IR (format of ir.py:1-8)."""
    mod: Module | None = None
    fn: Func | None = None
    blk: Block | None = None
    for no, raw in enumerate(text.splitlines(), 1):
        if not raw.strip():
            continue
        if raw.startswith("target "):
            mod = Module(raw[len("target "):].strip())
            continue
        if mod is None:
            raise RegionCompileError(f"line {no}: expected a target line first")
        if raw.startswith("global "):
            m = _GLOBAL_RE.match(raw)
            if not m:
                raise RegionCompileError(f"line {no}: malformed global")
            name, space, ty, count, init = m.groups()
            mod.globals.append(Global(name, space, ty, int(count),
                                      init if init in ("zero", "none") else int(init)))
            continue
        if raw.startswith("func "):
            m = _FUNC_RE.match(raw)
            if not m:
                raise RegionCompileError(f"line {no}: malformed function header")
            name, ptext, ret = m.groups()
            params = []
            for p in (ptext.split(", ") if ptext else []):
                pm = _PARAM_RE.match(p)
                if not pm:
                    raise RegionCompileError(f"line {no}: malformed parameter {p!r}")
                params.append((pm.group(1), pm.group(2)))
            fn = Func(name, params, None if ret == "void" else ret)
            blk = None
            continue
        if raw == "}":
            if fn is None:
                raise RegionCompileError(f"line {no}: stray '}}'")
            mod.funcs.append(fn)
            fn = None
            continue
        if fn is None:
            raise RegionCompileError(f"line {no}: unexpected line {raw!r}")
        lm = _LABEL_RE.match(raw)
        if lm:
            blk = Block(lm.group(1))
            fn.blocks.append(blk)
            continue
        sm = _SLOT_RE.match(raw)
        if sm and raw.lstrip().startswith("local "):
            name, count, aty, sty = sm.groups()
            fn.slots.append(Slot(name, aty or sty, int(count) if count else None))
            continue
        im = _INSTR_RE.match(raw)
        if not im or blk is None:
            raise RegionCompileError(f"line {no}: malformed instruction {raw.strip()!r}")
        dst, op, rest = im.groups()
        if op == "call":
            cm = _CALL_RE.match(rest or "")
            if not cm:
                raise RegionCompileError(f"line {no}: malformed call")
            args = [cm.group(1)] + ([a for a in cm.group(2).split(", ")] if cm.group(2) else [])
        else:
            args = rest.split(", ") if rest else []
        blk.instrs.append(Ins(op, dst, args))
    if mod is None:
        raise RegionCompileError("empty module")
    return mod


# ------------------------------------------------------------- layout (vgpu)

def _align(n: int) -> int:
    return (n + GLOBAL_ALIGN - 1) // GLOBAL_ALIGN * GLOBAL_ALIGN


def layout(mod: Module) -> tuple[list[dict], int, int]:
    """Offsets of every global in its space, as vgpu._layout (vgpu.py:171-207)."""
    out, gsize, ssize = [], 0, 0
    for g in mod.globals:
        extent = _SIZES[g.ty] * g.count
        if g.space == "team_shared":
            ssize = _align(ssize)
            off = ssize
            ssize += extent
        else:
            gsize = _align(gsize)
            off = gsize
            gsize += extent
        out.append({"name": g.name, "space": g.space, "ty": g.ty, "count": g.count,
                    "init": g.init, "off": off, "bytes": extent})
    return out, gsize, ssize


# ------------------------------------------------------------ translation

_ALU3 = {"add": "+", "sub": "-", "mul": "*"}
_BITW = {"and": "&", "or": "|", "xor": "^"}
_DIVS = {"udiv": 0, "urem": 1, "sdiv": 2, "srem": 3}
_CMP = {"eq": "==", "ne": "!=", "lt": "<", "le": "<=", "gt": ">", "ge": ">="}
_ATOMICS = {"add": 0, "max": 1, "min": 2, "xchg": 3, "cas": 4}
_QUERIES = {
    "__nvvm_read_ptx_sreg_tid": "threadIdx.x", "vgpu.thread.id": "threadIdx.x",
    "__nvvm_read_ptx_sreg_ctaid": "blockIdx.x", "vgpu.team.id": "blockIdx.x",
    "__nvvm_read_ptx_sreg_ntid": "blockDim.x", "vgpu.num.threads": "blockDim.x",
    "__nvvm_read_ptx_sreg_nctaid": "gridDim.x", "vgpu.num.teams": "gridDim.x",
}
_INC = ("__nvvm_atom_inc_gen_ui", "vgpu.atomic.inc")
_FENCE = ("__nvvm_membar_gl", "vgpu.fence")
_BARRIER = ("__nvvm_barrier0", "vgpu.barrier")
_TRAP = ("__nvvm_trap", "vgpu.trap")
SUPPORTED_TARGETS = ("nvptx64", "nvptx", "vgpu")


def _bits(ty: str) -> int:
    if ty not in _SIZES:
        raise RegionCompileError(f"unknown scalar type {ty!r}")
    return _SIZES[ty] * 8


def _lit(v: int, ty: str) -> str:
    return f"{v & ((1 << _bits(ty)) - 1)}ull"


class _Translator:
    def __init__(self, mod: Module):
        if mod.target not in SUPPORTED_TARGETS:
            raise RegionCompileError(f"image targets {mod.target!r}; the B200 backend "
                                     f"translates {', '.join(SUPPORTED_TARGETS)} images")
        self.mod = mod
        self.lay, self.gsize, self.ssize = layout(mod)
        self.gl = {g["name"]: g for g in self.lay}
        self.fnames = {f.name: f"f{k}" for k, f in enumerate(mod.funcs)}
        self.funcs = {f.name: f for f in mod.funcs}
        self.sites: list[dict] = []
        self.slot_labels: list[str] = []
        self.has_barrier = False
        self.kernels = [f for f in mod.funcs if f.name.startswith(KERNEL_PREFIX)]
        for k in self.kernels:
            if not re.fullmatch(r"[A-Za-z_]\w*", k.name):
                raise RegionCompileError(f"kernel name {k.name!r} is not an identifier")

    def site(self, **kw) -> int:
        self.sites.append(kw)
        return len(self.sites) - 1

    @staticmethod
    def _ctype(ty: str | None) -> str:
        if ty is None:
            return "void"
        return "P" if ty.startswith("ptr<") else "u64"

    def func(self, f: Func) -> tuple[str, str]:
        names: dict[str, str] = {}
        types: dict[str, str] = {}

        def vname(tok: str) -> str:
            if not tok.startswith("%"):
                raise RegionCompileError(f"@{f.name}: operand {tok!r} is not a value")
            key = tok[1:]
            if key not in names:
                raise RegionCompileError(f"@{f.name}: value {tok} used before definition")
            return names[key]

        params = ["u64 *__ic"]  # the thread's executed-instruction count
        for k, (pn, pt) in enumerate(f.params):
            names[pn] = f"a{k}"
            types[pn] = "P" if pt.startswith("ptr<") else "u64"
            params.append(f"{types[pn]} a{k}")
        slots = {}
        decl = []
        for k, s in enumerate(f.slots):
            ct = "u32" if _SIZES[s.ty] == 4 else "u64"
            n = s.count if s.count is not None else 1
            lab = len(self.slot_labels)
            self.slot_labels.append(f"slot:{s.name}")
            slots[s.name] = (f"s{k}", ct, n, _SIZES[s.ty] * n, lab)
            poison = "0xAAAAAAAAu" if ct == "u32" else "0xAAAAAAAAAAAAAAAAull"
            decl.append(f"  {ct} s{k}[{n}];")
            decl.append(f"  for (int i = 0; i < {n}; ++i) s{k}[i] = {poison};")
        # temporaries: one declaration each, typed by the producing op
        order = {b.label: i for i, b in enumerate(f.blocks)}
        tdecl = []
        for b in f.blocks:
            for ins in b.instrs:
                if ins.dst is None or ins.dst in names:
                    continue
                if ins.op in ("addr.slot", "addr.gv") or ins.op.startswith("elem.addr."):
                    t = "P"
                elif ins.op == "call":
                    callee = self.funcs.get(ins.args[0][1:])
                    if callee is None:
                        raise RegionCompileError(f"call to unknown function {ins.args[0]}")
                    t = self._ctype(callee.ret)
                else:
                    t = "u64"
                names[ins.dst] = f"t{len(tdecl)}"
                types[ins.dst] = t
                tdecl.append(f"  {t} t{len(tdecl)};")
        body = []
        for bi, b in enumerate(f.blocks):
            body.append(f"{b.label}:; *__ic += {len(b.instrs)}ull;")
            for ins in b.instrs:
                body.append("  " + self.instr(f, ins, vname, slots, order, bi))
        ret = self._ctype(f.ret)
        sig = f"__device__ {ret} {self.fnames[f.name]}({', '.join(params)})"
        text = "\n".join([sig + " {"] + decl + tdecl + body + ["}"])
        return sig + ";", text

    def instr(self, f: Func, ins: Ins, v, slots, order, bi) -> str:
        op, a = ins.op, ins.args
        parts = op.split(".")
        d = None
        if ins.dst is not None:
            d = v("%" + ins.dst)

        def put(expr: str) -> str:
            return f"{d} = {expr};" if d is not None else f"(void)({expr});"

        if op.startswith("const."):
            return put(_lit(int(a[0]), parts[1]))
        if len(parts) == 2 and parts[0] in _ALU3:
            return put(f"rt_mask({v(a[0])} {_ALU3[parts[0]]} {v(a[1])}, {_bits(parts[1])})")
        if len(parts) == 2 and parts[0] in _BITW:
            return put(f"({v(a[0])} {_BITW[parts[0]]} {v(a[1])})")
        if len(parts) == 2 and parts[0] in ("shl", "lshr", "ashr"):
            return put(f"rt_{parts[0]}({v(a[0])}, {v(a[1])}, {_bits(parts[1])})")
        if len(parts) == 2 and parts[0] == "neg":
            return put(f"rt_mask(0ull - {v(a[0])}, {_bits(parts[1])})")
        if len(parts) == 2 and parts[0] in _DIVS:
            s = self.site(kind="div", detail=f"{op} by zero")
            return put(f"rt_div({_DIVS[parts[0]]}, {v(a[0])}, {v(a[1])}, {_bits(parts[1])}, {s})")
        if parts[0] == "cmp" and len(parts) == 3:
            cc, ty = parts[1], parts[2]
            bits = _bits(ty)
            sgn = cc.startswith("s")
            base = cc[1:] if cc[0] in "su" else cc
            if base not in _CMP:
                raise RegionCompileError(f"unknown comparison {op}")
            if sgn:
                return put(f"(rt_sext({v(a[0])}, {bits}) {_CMP[base]} rt_sext({v(a[1])}, {bits}) ? 1ull : 0ull)")
            return put(f"({v(a[0])} {_CMP[base]} {v(a[1])} ? 1ull : 0ull)")
        if parts[0] == "cast" and len(parts) == 3:
            src, dst = parts[1], parts[2]
            return put(f"rt_cast({v(a[0])}, {_bits(src)}, {'true' if src in _SIGNED else 'false'}, {_bits(dst)})")
        if op in ("ld.slot", "st.slot", "addr.slot"):
            s = slots.get(a[0][1:])
            if s is None:
                raise RegionCompileError(f"@{f.name}: unknown slot {a[0]}")
            name, ct, n, nbytes, lab = s
            if op == "ld.slot":
                return put(f"(u64){name}[0]")
            if op == "st.slot":
                return f"{name}[0] = ({ct}){v(a[1])};"
            return put(f"rt_slot_ptr({name}, {nbytes}u, {lab}u)")
        if op == "addr.gv":
            g = self.gl.get(a[0][1:])
            if g is None:
                raise RegionCompileError(f"unknown global {a[0]}")
            fn = "rt_shared_ptr" if g["space"] == "team_shared" else "rt_global_ptr"
            return put(f"{fn}({g['off']}ull, {g['bytes']}u)")
        if parts[:2] == ["elem", "addr"] and len(parts) == 3:
            s = self.site(kind="elem")
            return put(f"rt_elem({v(a[0])}, {v(a[1])}, {_SIZES[parts[2]]}u, {s})")
        if parts[0] == "ld" and len(parts) == 2:
            s = self.site(kind="access", what="load")
            return put(f"rt_ld({v(a[0])}, {_SIZES[parts[1]]}u, {s})")
        if parts[0] == "st" and len(parts) == 2:
            s = self.site(kind="access", what="store")
            return f"rt_st({v(a[0])}, {_SIZES[parts[1]]}u, {v(a[1])}, {s});"
        if op == "call":
            callee = self.funcs.get(a[0][1:])
            if callee is None:
                raise RegionCompileError(f"call to unknown function {a[0]}")
            call = f"{self.fnames[callee.name]}({', '.join(['__ic'] + [v(x) for x in a[1:]])})"
            return f"{d} = {call};" if d is not None else f"{call};"
        if op == "ret":
            return f"return {v(a[0])};" if a else "return;"
        if op == "br":
            poll = "rt_poll(); " if order[a[0]] <= bi else ""
            return f"{poll}goto {a[0]};"
        if op == "cbr":
            pt = "rt_poll(); " if order[a[1]] <= bi else ""
            pf = "rt_poll(); " if order[a[2]] <= bi else ""
            return f"if ({v(a[0])}) {{ {pt}goto {a[1]}; }} else {{ {pf}goto {a[2]}; }}"
        if parts[0] == "atomic" and len(parts) == 4:
            kind, ty = parts[1], parts[3]
            if kind not in _ATOMICS:
                raise RegionCompileError(f"unknown atomic {op}")
            sl = self.site(kind="access", what="atomic load")
            ss = self.site(kind="access", what="atomic store")
            dd = v(a[2]) if kind == "cas" else "0ull"
            sgn = "true" if ty in _SIGNED else "false"
            return "rt_jitter(*__ic); " + put(f"rt_atomic({v(a[0])}, {_ATOMICS[kind]}u, {sgn}, {_SIZES[ty]}u, "
                       f"{v(a[1])}, {dd}, {sl}, {ss})")
        if op in _INC:
            sl = self.site(kind="access", what="atomic load")
            ss = self.site(kind="access", what="atomic store")
            return "rt_jitter(*__ic); " + put(
                f"rt_atomic({v(a[0])}, 5u, false, 4u, {v(a[1])}, 0ull, {sl}, {ss})")
        if op in _FENCE:
            return "__threadfence();"
        if op in _BARRIER:
            self.has_barrier = True
            s = self.site(kind="deadlock")
            return f"rt_jitter(*__ic); rt_barrier({s});"
        if op in _TRAP:
            s = self.site(kind="trap", func=f.name)
            c = v(a[0])
            return (f"rt_trap({c} == 1ull ? 1u : {c} == 2ull ? 2u : {c} == 3ull ? 3u : 8u, "
                    f"{s}, {c}, 0, 0, 0);")
        if op in _QUERIES:
            return put(f"(u64){_QUERIES[op]}")
        raise RegionCompileError(f"the B200 backend cannot translate opcode {op!r}")

    def kernel(self, k: Func) -> tuple[str, dict]:
        slots = ARGV_HEADER
        unpack = []
        args = []
        for pn, pt in k.params:
            if pt.startswith("ptr<"):
                unpack.append(f"  P p{len(args)} = rt_arg_ptr(a.v[{slots}], a.v[{slots + 1}], "
                              f"a.v[{slots + 2}]);")
                args.append(f"p{len(args)}")
                slots += 3
            else:
                bits = _bits(pt)
                unpack.append(f"  u64 p{len(args)} = rt_mask(a.v[{slots}], {bits});")
                args.append(f"p{len(args)}")
                slots += 1
        inits = []
        for g in self.lay:
            if g["space"] != "team_shared":
                continue
            kind = 2 if g["init"] == "none" else (0 if g["init"] == "zero" else 1)
            val = 0 if kind != 1 else int(g["init"]) & ((1 << _bits(g["ty"])) - 1)
            inits.append(f"  rt_shared_init({g['off']}ull, {g['bytes']}u, {kind}, {val}ull, "
                         f"{_SIZES[g['ty']]}u);")
        if k.ret is not None:
            raise RegionCompileError(f"kernel {k.name} returns a value")
        src = "\n".join(
            [f"struct A_{k.name} {{ u64 v[{slots}]; }};",
             f'extern "C" __global__ void __launch_bounds__(1024) {k.name}(const A_{k.name} a) {{',
             f"  rt_prologue(a.v, {self.ssize}u);"] + inits +
            ["  __syncthreads();"] + unpack +
            ["  u64 ic = 0;", f"  {self.fnames[k.name]}({', '.join(['&ic'] + args)});",
             "  rt_count(ic);", "  rt_finish();", "}"])
        return src, {"params": [list(p) for p in k.params], "argv_slots": slots}

    def translate(self) -> tuple[str, dict]:
        protos, bodies = [], []
        for f in self.mod.funcs:
            p, b = self.func(f)
            protos.append(p)
            bodies.append(b)
        kernels, kinfo = [], {}
        for k in self.kernels:
            s, info = self.kernel(k)
            kernels.append(s)
            kinfo[k.name] = info
        prelude = (CSRC / "region_rt.cuh").read_text()
        src = "\n\n".join([prelude, "\n".join(protos)] + bodies + kernels) + "\n"
        manifest = {
            "format": 1, "arch": ARCH, "source_target": self.mod.target,
            "kernels": kinfo, "globals": self.lay, "global_bytes": self.gsize,
            "shared_bytes": self.ssize, "sites": self.sites, "slot_labels": self.slot_labels,
            "has_barrier": self.has_barrier,
            "functions": [f.name for f in self.mod.funcs],
        }
        return src, manifest


def translate(ir_text: str) -> tuple[str, dict]:
    """IR text -> (CUDA C++ source, manifest)."""
    return _Translator(parse_ir(ir_text)).translate()


# ------------------------------------------------------------------ NVRTC

_nvrtc = None


def _load_nvrtc():
    global _nvrtc
    if _nvrtc is not None:
        return _nvrtc
    cands = [os.environ.get("OMPRT_NVRTC", ""), "/usr/local/cuda/lib64/libnvrtc.so.12",
             "/usr/local/cuda/lib64/libnvrtc.so", ctypes.util.find_library("nvrtc") or ""]
    try:
        import nvidia.cuda_nvrtc as _pkg  # the wheel torch depends on

        for d in _pkg.__path__:
            cands += [str(p) for p in sorted(Path(d).glob("lib/libnvrtc.so*"))]
    except ImportError:
        pass
    for c in cands:
        if c and os.path.exists(c) or (c and "/" not in c):
            try:
                lib = ctypes.CDLL(c)
                break
            except OSError:
                continue
    else:
        raise RegionCompileError("libnvrtc not found (set OMPRT_NVRTC)")
    lib.nvrtcGetErrorString.restype = ctypes.c_char_p
    _nvrtc = lib
    return lib


def _check(lib, rc, what):
    if rc != 0:
        raise RegionCompileError(f"{what}: {lib.nvrtcGetErrorString(rc).decode()}")


def nvrtc_compile(src: str, name: str = "region.cu", lineinfo: bool = True) -> bytes:
    """CUDA C++ -> sm_100a cubin with NVRTC."""
    lib = _load_nvrtc()
    prog = ctypes.c_void_p()
    _check(lib, lib.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), name.encode(),
                                       0, None, None), "nvrtcCreateProgram")
    opts = [f"--gpu-architecture={ARCH}", "-std=c++17", "-default-device", "--device-int128",
            "-diag-suppress=177,550"]
    if lineinfo:
        opts.append("-lineinfo")
    arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
    try:
        rc = lib.nvrtcCompileProgram(prog, len(opts), arr)
        n = ctypes.c_size_t()
        lib.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
        log = ctypes.create_string_buffer(n.value)
        lib.nvrtcGetProgramLog(prog, log)
        if rc != 0:
            raise RegionCompileError(f"NVRTC: {lib.nvrtcGetErrorString(rc).decode()}\n"
                                     f"{log.value.decode(errors='replace')}")
        _check(lib, lib.nvrtcGetCUBINSize(prog, ctypes.byref(n)), "nvrtcGetCUBINSize")
        buf = ctypes.create_string_buffer(n.value)
        _check(lib, lib.nvrtcGetCUBIN(prog, buf), "nvrtcGetCUBIN")
        return buf.raw
    finally:
        lib.nvrtcDestroyProgram(ctypes.byref(prog))


def nvrtc_version() -> str:
    lib = _load_nvrtc()
    a, b = ctypes.c_int(), ctypes.c_int()
    lib.nvrtcVersion(ctypes.byref(a), ctypes.byref(b))
    return f"{a.value}.{b.value}"


# ------------------------------------------------------------------ images

@dataclass
class B200Image:
    """A compiled device image: manifest + sm_100a cubin."""

    manifest: dict
    cubin: bytes

    @property
    def kernels(self) -> dict:
        return self.manifest["kernels"]

    def to_bytes(self) -> bytes:
        m = json.dumps(self.manifest, sort_keys=True).encode()
        return (IMAGE_MAGIC + struct.pack("<I", len(m)) + m + struct.pack("<Q", len(self.cubin))
                + self.cubin)

    @classmethod
    def from_bytes(cls, data: bytes) -> "B200Image":
        data = bytes(data)
        if data[:8] != IMAGE_MAGIC:
            raise BadImage(f"expected magic {IMAGE_MAGIC!r}")
        try:
            (ml,) = struct.unpack_from("<I", data, 8)
            manifest = json.loads(data[12:12 + ml].decode())
            (cl,) = struct.unpack_from("<Q", data, 12 + ml)
        except (struct.error, ValueError, UnicodeDecodeError) as e:
            raise BadImage(f"malformed B200 image: {e}") from None
        start = 20 + ml
        if start + cl != len(data):
            raise BadImage("B200 image length fields do not match its size")
        if manifest.get("format") != 1 or manifest.get("arch") != ARCH:
            raise BadImage(f"unsupported B200 image format/arch "
                           f"{manifest.get('format')}/{manifest.get('arch')}")
        return cls(manifest, data[start:])


_CACHE: dict[str, B200Image] = {}


def compile_image(ir_text: str) -> B200Image:
    """IR image text (nvptx64 or vgpu target) -> B200Image (cached by IR hash)."""
    key = hashlib.sha256(ir_text.encode()).hexdigest()
    img = _CACHE.get(key)
    if img is None:
        src, manifest = translate(ir_text)
        manifest["ir_sha256"] = key
        manifest["nvrtc"] = nvrtc_version()
        img = B200Image(manifest, nvrtc_compile(src))
        _CACHE[key] = img
    return img
