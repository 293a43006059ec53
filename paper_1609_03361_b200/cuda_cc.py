"""sf-cuda-cc — a C-compiler stand-in that runs the reference's JIT'd kernels on
the B200.

The reference (stencilforge) JIT-compiles every Operator by writing C99 and
invoking `<cc> -std=c99 -O3 ... -shared -o kernel.so kernel.c -lm`
(jit.cpp:67-80), where <cc> is $STENCILFORGE_CC, CodegenConfig::cc_override or
the preset (jit.cpp:84-95), then dlsym()s `Operator` and calls it with the
GridFunction host pointers (jit.cpp:104-148). Pointing STENCILFORGE_CC at this
tool (bin/sf-cuda-cc) moves every operator the unmodified reference builds onto
the GPU, with the same ABI and the same bitwise results:

* recognised operators — the acoustic forward/adjoint update (2D/3D, any
  order, with its injection and sampling loops) and the diffusion update —
  are lifted from the generated source (shapes, step count, direction, point
  counts and every folded fp32 literal exactly as printed) and bound to the
  tuned kernels of libsf_b200.so (sf_acoustic_plan_create_ex /
  sf_diffusion_plan_create_ex);
* any other operator is translated statement for statement into CUDA
  (one kernel per parallel loop nest, thread-per-point; each `omp single`
  loop a single-thread kernel so its sequential order is kept; time-slot
  aliases computed on the host) and built with nvcc for sm_100a with
  --fmad=false, so every expression rounds exactly as gcc -ffp-contract=off
  evaluates it.

Either way the produced shared library exports `int Operator(...)` taking the
same host pointers; it uploads, runs all steps, downloads, and returns 0.
"""
from __future__ import annotations

import os
import re
import subprocess
import sys
import tempfile
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("SF_NVCC", "/usr/local/cuda/bin/nvcc")


class Unsupported(Exception):
    pass


# ---------------------------------------------------------------------------
# parsing the generated translation unit (codegen.cpp:411-502)

@dataclass
class Array:
    name: str
    ctype: str          # float / double / int
    dims: list          # trailing extents from the cast; [] for 1-D


@dataclass
class Node:
    kind: str                          # loop / single / aliases / assign / decl
    pragma: str = ""
    var: str = ""
    lo: str = ""
    hi: str = ""
    step: int = 1
    descending: bool = False
    body: list = field(default_factory=list)
    text: str = ""                     # assign/decl statement (without ';')
    aliases: list = field(default_factory=list)  # (name, offset, modulus)


@dataclass
class Program:
    entry: str
    params: list        # (ctype, name_vec)
    arrays: dict        # name -> Array
    alias_names: list
    roots: list


LOOP_RE = re.compile(r"^for \(int (\w+) = (.+?); \1 (<|>=) (.+?); \1 ([+-])= (\d+)\)$")
CAP_RE = re.compile(r"^const int (\w+)_hi = \((\w+) \+ (\d+) < (\w+)\) \? \2 \+ \3 : \4;$")
ALIAS_RE = re.compile(r"^(t\d+) = \((\w+)(?: \+ (\d+))?\) % (\d+);$")


def parse(src: str) -> Program:
    lines = [ln.strip() for ln in src.splitlines()]
    lines = [ln for ln in lines if ln and not ln.startswith("#include")]
    pos = 0
    m = re.match(r"^int (\w+)\((.*)\)$", lines[pos])
    if not m:
        raise Unsupported("no entry signature")
    entry = m.group(1)
    params = []
    for part in m.group(2).split(", "):
        pm = re.match(r"^(float|double|int) \*(\w+)_vec$", part)
        if not pm:
            raise Unsupported(f"parameter {part!r}")
        params.append((pm.group(1), pm.group(2)))
    pos += 1
    if lines[pos] != "{":
        raise Unsupported("body")
    pos += 1
    arrays = {}
    while True:
        ln = lines[pos]
        am = re.match(r"^(float|double|int) \(\*(\w+)\)((?:\[\d+\])+) = .*\) \2_vec;$", ln)
        bm = re.match(r"^(float|double|int) \*(\w+) = \2_vec;$", ln)
        if am:
            arrays[am.group(2)] = Array(am.group(2), am.group(1),
                                        [int(x) for x in re.findall(r"\[(\d+)\]", am.group(3))])
        elif bm:
            arrays[bm.group(2)] = Array(bm.group(2), bm.group(1), [])
        else:
            break
        pos += 1
    if lines[pos] != "{":
        raise Unsupported("inner block")
    pos += 1
    alias_names = []
    while re.match(r"^int t\d+;$", lines[pos]):
        alias_names.append(lines[pos][4:-1])
        pos += 1
    if lines[pos] == "#pragma omp parallel":
        pos += 1

    def parse_block(pos):
        """parse statements until the matching '}' (pos at first line after '{')."""
        nodes = []
        pragma = ""
        while True:
            ln = lines[pos]
            if ln == "}":
                return nodes, pos + 1
            if ln.startswith("#pragma"):
                pragma = ln
                pos += 1
                continue
            lm = LOOP_RE.match(ln)
            if lm:
                var, lo, cmp, hi, sign, step = lm.groups()
                if lines[pos + 1] != "{":
                    raise Unsupported("loop without block")
                body, pos = parse_block(pos + 2)
                nodes.append(Node("loop", pragma, var, lo, hi, int(step), cmp == ">=", body))
                pragma = ""
                continue
            if ln == "{":
                # alias block (omp single) or a plain block
                body_start = pos + 1
                als = []
                q = body_start
                while ALIAS_RE.match(lines[q]):
                    am = ALIAS_RE.match(lines[q])
                    als.append((am.group(1), int(am.group(3) or 0), int(am.group(4))))
                    q += 1
                if als and lines[q] == "}":
                    nodes.append(Node("aliases", pragma, aliases=als))
                    pos = q + 1
                else:
                    body, pos = parse_block(pos + 1)
                    nodes.extend(body)
                pragma = ""
                continue
            cm = CAP_RE.match(ln)
            if cm:
                # remainder bound of a blocked loop (codegen.cpp:291-300)
                nodes.append(Node("cap", var=cm.group(1), lo=cm.group(2), hi=cm.group(4),
                                  step=int(cm.group(3))))
                pos += 1
                continue
            if ln.endswith(";"):
                kind = "decl" if ln.startswith("const ") else "assign"
                nodes.append(Node(kind, text=ln[:-1]))
                pos += 1
                continue
            raise Unsupported(f"line {ln!r}")

    if LOOP_RE.match(lines[pos]) or lines[pos] == "{":
        roots, pos = parse_block_top(lines, pos, parse_block)
    else:
        raise Unsupported("no loop nest")
    return Program(entry, params, arrays, alias_names, unblock(roots))


def _caps(nodes):
    for n in nodes:
        if n.kind == "cap":
            yield n
        yield from _caps(n.body)


def _rebound(nodes, var, bvar, lo, hi, size):
    """Give loop `var` (lo = bvar, hi = var_hi) the block loop's full range and
    drop its cap."""
    out = []
    for n in nodes:
        if n.kind == "cap" and n.var == var:
            if n.lo != bvar or n.hi != hi or n.step != size:
                raise Unsupported("cap")
            continue
        if n.kind == "loop":
            n.body = _rebound(n.body, var, bvar, lo, hi, size)
            if n.var == var:
                if n.lo != bvar or n.hi != f"{var}_hi" or n.step != 1:
                    raise Unsupported("blocked loop bounds")
                n.lo, n.hi = lo, hi
        out.append(n)
    return out


def unblock(nodes):
    """Undo loop blocking (opt.cpp:136-200): a block loop `for (vb = lo; vb < hi;
    vb += S)` over `for (v = vb; v < min(vb + S, hi); ...)` visits exactly the
    points of `for (v = lo; v < hi; ...)`, and the reference only blocks
    parallelisable dimensions (opt.cpp:167-169), whose points are independent;
    the GPU schedule is chosen here instead."""
    out = []
    for n in nodes:
        if n.kind == "loop":
            n.body = unblock(n.body)
            caps = [c for c in _caps(n.body) if c.lo == n.var]
            if caps:
                if len(caps) != 1 or n.descending or n.step != caps[0].step:
                    raise Unsupported("block loop")
                out.extend(_rebound(n.body, caps[0].var, n.var, n.lo, n.hi, n.step))
                continue
        out.append(n)
    return out


def parse_block_top(lines, pos, parse_block):
    # the root is either one loop or a braced block of nodes; parse_block
    # stops at the closing brace of the enclosing "{ int t0; ... }" block
    nodes, pos = parse_block(pos)
    return nodes, pos


# ---------------------------------------------------------------------------
# recognising the reference's own operators

TERM_SPLIT = re.compile(r"\s([+-])\s")


def split_terms(rhs: str):
    """Top-level ' + ' / ' - ' split of an emitted expression."""
    terms, depth, cur, sign = [], 0, "", "+"
    i = 0
    if rhs.startswith("-"):
        sign, i = "-", 1
    while i < len(rhs):
        ch = rhs[i]
        if ch in "[(":
            depth += 1
        elif ch in "])":
            depth -= 1
        if depth == 0 and (rhs.startswith(" + ", i) or rhs.startswith(" - ", i)):
            terms.append((sign, cur))
            sign = rhs[i + 1]
            cur = ""
            i += 3
            continue
        cur += ch
        i += 1
    terms.append((sign, cur))
    return terms


def lit(s: str) -> float:
    if not re.match(r"^[0-9.]+e-?\d+F$", s):
        raise Unsupported(f"literal {s!r}")
    return float(np.float32(float(s[:-1])))


def offsets(idx: str, loopvars):
    """'[i1][i2 - 2][i3]' -> [0, -2, 0] (checking the loop variables)."""
    parts = re.findall(r"\[([^\]]+)\]", idx)
    out = []
    for part, var in zip(parts, loopvars):
        m = re.match(rf"^{var}(?: ([+-]) (\d+))?$", part.strip())
        if not m:
            raise Unsupported(f"index {part!r}")
        out.append(0 if m.group(1) is None else int(m.group(2)) * (1 if m.group(1) == "+" else -1))
    if len(parts) != len(loopvars):
        raise Unsupported("index rank")
    return out


def nest_of(loop: Node):
    """[(var, lo, hi)], innermost body of a perfect loop nest."""
    levels = []
    node = loop
    while True:
        if node.kind != "loop" or node.step != 1 or node.descending:
            raise Unsupported("nest shape")
        levels.append((node.var, int(node.lo), int(node.hi)))
        if len(node.body) == 1 and node.body[0].kind == "loop":
            node = node.body[0]
            continue
        return levels, node.body


@dataclass
class AcousticOp:
    forward: bool
    field: str
    shape: tuple
    order: int
    nt: int
    n_src: int
    n_rec: int
    constants: list
    tsel: list


@dataclass
class DiffusionOp:
    shape: tuple
    order: int
    nt: int
    c0: float
    has_c0: bool
    cj: list


def recognise(prog: Program):
    roots = prog.roots
    if len(roots) != 1 or roots[0].kind != "loop":
        return None
    tl = roots[0]
    body = tl.body
    if not body or body[0].kind != "aliases":
        return None
    aliases = {name: (off, mod) for name, off, mod in body[0].aliases}
    tvar = tl.var
    try:
        if len(aliases) == 3:
            return recognise_acoustic(prog, tl, aliases, tvar)
        if len(aliases) == 2 and len(body) == 2:
            return recognise_diffusion(prog, tl, aliases, tvar)
    except Unsupported:
        return None
    return None


def recognise_diffusion(prog, tl, aliases, tvar):
    if tl.descending or tl.lo != "0":
        raise Unsupported("diffusion loop")
    nt = int(tl.hi)
    if aliases != {"t0": (0, 2), "t1": (1, 2)}:
        raise Unsupported("aliases")
    levels, inner = nest_of(tl.body[1])
    if len(levels) != 2 or len(inner) != 1 or inner[0].kind != "assign":
        raise Unsupported("diffusion nest")
    field = [a for a in prog.arrays.values() if len(a.dims) == 2]
    if len(prog.params) != 1 or len(field) != 1 or field[0].ctype != "float":
        raise Unsupported("diffusion args")
    u = field[0]
    nx, ny = int(levels[0][2]) + levels[0][1], int(levels[1][2]) + levels[1][1]
    if [nx, ny] != u.dims:
        raise Unsupported("diffusion shape")
    r = levels[0][1]
    lhs, rhs = inner[0].text.split(" = ", 1)
    if lhs != f"{u.name}[t1][{levels[0][0]}][{levels[1][0]}]":
        raise Unsupported("lhs")
    vars_ = [levels[0][0], levels[1][0]]
    terms = []
    for sign, body in split_terms(rhs):
        f = body.split("*")
        if len(f) == 1:
            c, ref = 1.0, f[0]
        elif len(f) == 2:
            c, ref = lit(f[0]), f[1]
        else:
            raise Unsupported("term")
        if sign == "-":
            c = -c
        m = re.match(rf"^{u.name}\[t0\]((?:\[[^\]]+\])+)$", ref)
        if not m:
            raise Unsupported("ref")
        terms.append((c, offsets(m.group(1), vars_)))
    expect = []
    has_c0 = terms and terms[0][1] == [0, 0]
    if has_c0:
        expect.append([0, 0])
    for axis in (1, 0):
        for j in list(range(-r, 0)) + list(range(1, r + 1)):
            o = [0, 0]
            o[axis] = j
            expect.append(o)
    if [t[1] for t in terms] != expect:
        raise Unsupported("term order")
    cj = [0.0] * 8
    nb = terms[1:] if has_c0 else terms
    for (c, o) in nb:
        j = abs(o[0] + o[1])
        if cj[j - 1] == 0.0:
            cj[j - 1] = c
        elif np.float32(cj[j - 1]) != np.float32(c):
            raise Unsupported("asymmetric coefficients")
    return DiffusionOp((nx, ny), 2 * r, nt, terms[0][0] if has_c0 else 0.0, bool(has_c0), cj)


def recognise_acoustic(prog, tl, aliases, tvar):
    if aliases != {"t0": (2, 3), "t1": (0, 3), "t2": (1, 3)}:
        raise Unsupported("aliases")
    forward = not tl.descending
    if forward:
        if tl.lo != "0":
            raise Unsupported("time loop")
        nt = int(tl.hi)
    else:
        if tl.hi != "1":
            raise Unsupported("time loop")
        nt = int(tl.lo)
    if nt < 1:
        raise Unsupported("no time steps")
    body = tl.body
    if len(body) != 4 or any(b.kind != "loop" for b in body[1:]):
        raise Unsupported("acoustic structure")
    levels, inner = nest_of(body[1])
    ndim = len(levels)
    if ndim not in (2, 3) or len(inner) != 5:
        raise Unsupported("acoustic nest")
    fname = "u" if forward else "v"
    names = [p[1] for p in prog.params]
    if names != [fname, "m", "eta", "src", "src_ci", "src_w", "rec", "rec_ci", "rec_w"]:
        raise Unsupported("signature")
    if any(prog.arrays[n].ctype != ("int" if n.endswith("_ci") else "float") for n in names):
        raise Unsupported("element types")
    u = prog.arrays[fname]
    shape = tuple(u.dims)
    r = levels[0][1]
    if len(shape) != ndim or any(lo != r or hi != n - r for (v, lo, hi), n in zip(levels, shape)):
        raise Unsupported("bounds")
    vars_ = [lv[0] for lv in levels]
    idx = "".join(f"[{v}]" for v in vars_)
    # temps (op.cpp:28-51 CSE): ce*eta, cm*m, sum, reciprocal
    t = [n.text for n in inner[:4]]
    m0 = re.match(rf"^const float temp0 = ([^*]+)\*eta{re.escape(idx)}$", t[0])
    m1 = re.match(rf"^const float temp1 = ([^*]+)\*m{re.escape(idx)}$", t[1])
    if not (m0 and m1 and t[2] == "const float temp2 = temp0 + temp1"
            and t[3] == "const float temp3 = 1.0F/temp2"):
        raise Unsupported("temps")
    ce, cm = lit(m0.group(1)), lit(m1.group(1))
    out_alias = "t2" if forward else "t0"
    prev_alias = "t0" if forward else "t2"
    lhs, rhs = inner[4].text.split(" = ", 1)
    if lhs != f"{fname}[{out_alias}]{idx}":
        raise Unsupported("lhs")
    terms = split_terms(rhs)
    tc, tsel = [], []
    for sign, bodyt in terms[:3]:
        f = bodyt.split("*")
        if len(f) != 4 or f[1] != "temp3":
            raise Unsupported("time term")
        fld = f[2].split("[")[0]
        lv = re.match(rf"^{fname}\[(t\d)\]{re.escape(idx)}$", f[3])
        if fld not in ("eta", "m") or f[2] != fld + idx or not lv:
            raise Unsupported("time term refs")
        level = 0 if lv.group(1) == prev_alias else (1 if lv.group(1) == "t1" else -1)
        if level < 0:
            raise Unsupported("time level")
        tc.append(lit(f[0]) * (-1 if sign == "-" else 1))
        tsel.append(2 * (fld == "m") + level)
    rest = []
    for sign, bodyt in terms[3:]:
        f = bodyt.split("*")
        if len(f) != 3 or f[1] != "temp3":
            raise Unsupported("space term")
        rm = re.match(rf"^{fname}\[t1\]((?:\[[^\]]+\])+)$", f[2])
        if not rm:
            raise Unsupported("space ref")
        rest.append((lit(f[0]) * (-1 if sign == "-" else 1), offsets(rm.group(1), vars_)))
    expect = [[0] * ndim]
    for axis in reversed(range(ndim)):
        for j in list(range(-r, 0)) + list(range(1, r + 1)):
            o = [0] * ndim
            o[axis] = j
            expect.append(o)
    if [o for _, o in rest] != expect:
        raise Unsupported("space term order")
    c0 = rest[0][0]
    cj = [None] * r
    for c, o in rest[1:]:
        j = abs(sum(o))
        if cj[j - 1] is None:
            cj[j - 1] = c
        elif np.float32(cj[j - 1]) != np.float32(c):
            raise Unsupported("anisotropic coefficients")
    # sparse loops: injection then sampling, the expected sets and rows
    inj_set, smp_set = ("src", "rec") if forward else ("rec", "src")
    row = tvar if forward else f"{tvar} - 1"
    inj, smp = body[2], body[3]
    corners = 1 << ndim
    if len(inj.body) != corners or len(smp.body) != 1:
        raise Unsupported("sparse loops")
    def corner(pset, k):
        return "".join(f"[{pset}_ci[p][{d}]" + (" + 1" if (k >> d) & 1 else "") + "]"
                       for d in range(ndim))

    scale = None
    for k, st in enumerate(inj.body):
        at = f"{fname}[{out_alias}]{corner(inj_set, k)}"
        pre = f"{at} = "
        post = f"*{inj_set}[{row}][p]*{inj_set}_w[p][{k}]/m{corner(inj_set, k)} + {at}"
        if not (st.text.startswith(pre) and st.text.endswith(post)):
            raise Unsupported("injection")
        c = lit(st.text[len(pre):-len(post)])
        if scale is None:
            scale = c
        elif c != scale:
            raise Unsupported("injection scale")
    want = f"{smp_set}[{row}][p] = " + " + ".join(
        f"{smp_set}_w[p][{k}]*{fname}[{out_alias}]{corner(smp_set, k)}" for k in range(corners))
    if smp.body[0].text != want:
        raise Unsupported("sampling")
    n_src = prog.arrays["src"].dims[0]
    n_rec = prog.arrays["rec"].dims[0]
    if int(inj.hi) != (n_src if forward else n_rec) or int(smp.hi) != (n_rec if forward else n_src):
        raise Unsupported("point counts")
    consts = [ce, cm] + tc + [c0] + [cj[j] if j < r else 0.0 for j in range(8)] + [scale]
    return AcousticOp(forward, fname, shape, 2 * r, nt, n_src, n_rec, consts, tsel)


# ---------------------------------------------------------------------------
# code emission

def fmt(x: float) -> str:
    return repr(float(np.float32(x))) + "f" if np.isfinite(x) else "0.0f"


def emit_acoustic(op: AcousticOp, entry: str) -> str:
    shape = list(op.shape) + [1] * (3 - len(op.shape))
    consts = ", ".join(f"{float(np.float32(c))!r}f" for c in op.constants)
    return f"""// generated by sf-cuda-cc: the reference's acoustic operator bound to libsf_b200
#include "sf_b200.h"
static sf_plan* g_plan = 0;
extern "C" int {entry}(float* u, float* m, float* eta, float* src, int* src_ci, float* src_w,
                       float* rec, int* rec_ci, float* rec_w) {{
    if (!g_plan) {{
        sf_acoustic_desc d = {{}};
        d.ndim = {len(op.shape)};
        d.shape[0] = {shape[0]}; d.shape[1] = {shape[1]}; d.shape[2] = {shape[2]};
        d.space_order = {op.order};
        d.forward = {int(op.forward)};
        d.nt = {op.nt};
        d.dt = 1.0;        /* constants supplied below, as printed in the source */
        d.spacing = 1.0;
        d.n_src = {op.n_src};
        d.n_rec = {op.n_rec};
        const float c[15] = {{{consts}}};
        const int sel[3] = {{{", ".join(str(x) for x in op.tsel)}}};
        if (sf_acoustic_plan_create_ex(&d, c, sel, 0, &g_plan) != 0) return 1;
    }}
    return sf_acoustic_apply(g_plan, u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w);
}}
"""


def emit_diffusion(op: DiffusionOp, entry: str) -> str:
    cj = ", ".join(f"{float(np.float32(c))!r}f" for c in op.cj)
    return f"""// generated by sf-cuda-cc: the reference's diffusion operator bound to libsf_b200
#include "sf_b200.h"
static sf_plan* g_plan = 0;
extern "C" int {entry}(float* u) {{
    if (!g_plan) {{
        sf_diffusion_desc d = {{}};
        d.nx = {op.shape[0]}; d.ny = {op.shape[1]};
        d.order = {op.order};
        d.nt = {op.nt};
        d.alpha_num = d.alpha_den = d.dx_num = d.dx_den = 1;
        const float cj[8] = {{{cj}}};
        if (sf_diffusion_plan_create_ex(&d, {float(np.float32(op.c0))!r}f, {int(op.has_c0)}, cj, 0,
                                        &g_plan) != 0) return 1;
    }}
    return sf_diffusion_apply(g_plan, u);
}}
"""


def array_refs(text: str):
    """[(name, [subscript, ...])] for every `name[..][..]` in an expression."""
    out = []
    for m in re.finditer(r"\b([A-Za-z_]\w*)\[", text):
        if m.start() > 0 and text[m.start() - 1] in "]":
            continue
        name, i, subs = m.group(1), m.end() - 1, []
        while i < len(text) and text[i] == "[":
            depth, j = 0, i
            while True:
                depth += {"[": 1, "]": -1}.get(text[j], 0)
                if depth == 0:
                    break
                j += 1
            subs.append(text[i + 1:j].strip())
            i = j + 1
        out.append((name, subs))
    return out


def _statements(nodes):
    for n in nodes:
        if n.kind in ("assign", "decl"):
            yield n
        yield from _statements(n.body)


def _loop_vars(node):
    while node.kind == "loop":
        yield node.var
        node = node.body[0] if len(node.body) == 1 else Node("leaf")


def parallel_safe(nest: Node, aliases) -> bool:
    """Whether every point of a perfect loop nest can run concurrently.

    Conservative dependence test on the statement text: each written array
    element must be addressed injectively by the nest's variables (`v`, `v±c`,
    host-fixed scalars, literals — no indirection, so the sequential injection
    loops, whose corners may collide, stay sequential), and every read of a
    written array must be the same element or a different time slot (distinct
    modulo aliases of one alias block, codegen.cpp:336-354)."""
    try:
        levels, inner = nest_of(nest)
    except (Unsupported, ValueError):
        return False
    vars_ = {v for v, _, _ in levels}
    if any(n.kind not in ("assign", "decl") for n in inner):
        return False
    writes = {}
    for st in inner:
        if st.kind != "assign":
            continue
        lhs = st.text.split(" = ", 1)[0]
        refs = array_refs(lhs)
        if len(refs) != 1 or refs[0][0] + "".join(f"[{x}]" for x in refs[0][1]) != lhs:
            return False
        name, subs = refs[0]
        used = []
        for sub in subs:
            m = re.match(r"^(\w+)(?: [+-] \d+)?$", sub)
            if not m:
                return False
            if m.group(1) in vars_:
                used.append(m.group(1))
        if sorted(used) != sorted(vars_):
            return False
        if writes.setdefault(name, subs) != subs:
            return False
    def distinct(a, b):
        # provably different elements: some subscript pair differs by a
        # non-zero constant on the same loop-invariant base, or names two
        # different time slots of one alias block
        for x, y in zip(a, b):
            if x in aliases and y in aliases:
                if x != y:
                    return True
                continue
            mx = re.match(r"^(\w+)(?: ([+-]) (\d+))?$", x)
            my = re.match(r"^(\w+)(?: ([+-]) (\d+))?$", y)
            if not (mx and my):
                continue
            if mx.group(1) in vars_ or my.group(1) in vars_:
                continue
            ox = int(mx.group(3) or 0) * (-1 if mx.group(2) == "-" else 1)
            oy = int(my.group(3) or 0) * (-1 if my.group(2) == "-" else 1)
            if mx.group(1).isdigit() and my.group(1).isdigit():
                if int(mx.group(1)) + ox != int(my.group(1)) + oy:
                    return True
            elif mx.group(1) == my.group(1) and ox != oy:
                return True
        return False

    for st in inner:
        rhs = st.text.split(" = ", 1)[1]
        for name, subs in array_refs(rhs):
            if name not in writes or subs == writes[name]:
                continue
            if distinct(subs, writes[name]):
                continue
            return False
    return True


def emit_generic(prog: Program) -> str:
    """Statement-for-statement CUDA translation of the generated nest.

    Host-level structure (time loop, alias block, any loop that is not a
    parallel nest but holds loops) runs on the host, in order, on one stream;
    each parallel-safe perfect nest becomes one thread-per-point kernel; any
    other loop (the `omp single` injection/sampling loops, recurrences) runs in
    a one-thread kernel so its sequential order is kept."""
    arr_decl = []
    for ctype, name in prog.params:
        a = prog.arrays[name]
        if a.dims:
            dims = "".join(f"[{d}]" for d in a.dims)
            arr_decl.append(f"    {ctype} (*{name}){dims} = ({ctype} (*){dims}) {name}_vec;")
        else:
            arr_decl.append(f"    {ctype} *{name} = {name}_vec;")
    decls = "\n".join(arr_decl)
    params_dev = ", ".join(f"{c} *{n}_vec" for c, n in prog.params)
    args_dev = ", ".join(f"d_{n}" for _, n in prog.params)
    aliases = set(prog.alias_names)
    kernels, host = [], []

    def stmts(nodes, indent):
        out = []
        for n in nodes:
            if n.kind in ("assign", "decl"):
                out.append(" " * indent + n.text + ";")
            elif n.kind == "loop":
                cmp = ">=" if n.descending else "<"
                op_ = "-=" if n.descending else "+="
                out.append(" " * indent + f"for (int {n.var} = {n.lo}; {n.var} {cmp} {n.hi}; "
                           f"{n.var} {op_} {n.step}) {{")
                out.extend(stmts(n.body, indent + 4))
                out.append(" " * indent + "}")
            else:
                raise Unsupported(f"node {n.kind} inside a kernel")
        return out

    def launch(node_list, scalars, parallel):
        k = len(kernels)
        scalars = list(prog.alias_names) + list(scalars)
        sc = [f"int {v}" for v in scalars]
        sig = ", ".join([params_dev] + sc)
        call_args = ", ".join([args_dev] + list(scalars))
        if not parallel:
            body = "\n".join(stmts(node_list, 8))
            kernels.append(f"__global__ void sfk{k}({sig}) {{\n{decls}\n    {{\n{body}\n    }}\n}}")
            return f"sfk{k}<<<1, 1>>>({call_args});"
        levels, inner = nest_of(node_list[0])
        axes = ["x", "y", "z"]
        lines, conds = [], []
        for depth, (var, lo, hi) in enumerate(reversed(levels)):
            ax = axes[depth]
            lines.append(f"    const int {var} = {lo} + (int)(blockIdx.{ax} * blockDim.{ax} + threadIdx.{ax});")
            conds.append(f"{var} < {hi}")
        body = "\n".join(stmts(inner, 8))
        kernels.append(f"__global__ void sfk{k}({sig}) {{\n{decls}\n" + "\n".join(lines)
                       + f"\n    if ({' && '.join(conds)}) {{\n{body}\n    }}\n}}")
        ext = [hi - lo for _, lo, hi in reversed(levels)] + [1] * (3 - len(levels))
        block = {1: [256, 1, 1], 2: [32, 8, 1], 3: [32, 4, 2]}[len(levels)]
        grid = ", ".join(f"{(e + b - 1) // b}" for e, b in zip(ext, block))
        if any(e <= 0 for e in ext):
            return ";  /* empty nest */"
        return f"sfk{k}<<<dim3({grid}), dim3({block[0]}, {block[1]}, {block[2]})>>>({call_args});"

    def walk(nodes, scalars, indent):
        pad = " " * indent
        for n in nodes:
            if n.kind == "aliases":
                tv = scalars[-1] if scalars else None
                for name, off, mod in n.aliases:
                    if tv is None:
                        raise Unsupported("alias block outside a loop")
                    rhs = f"({tv} + {off}) % {mod}" if off else f"({tv}) % {mod}"
                    host.append(pad + f"{name} = {rhs};")
            elif n.kind == "loop":
                try:
                    levels, _ = nest_of(n)
                    nested_ok = len(levels) <= 3
                except (Unsupported, ValueError):
                    nested_ok = False
                if nested_ok and parallel_safe(n, aliases):
                    host.append(pad + launch([n], scalars, True))
                elif any(c.kind in ("loop", "aliases") for c in n.body):
                    cmp = ">=" if n.descending else "<"
                    op_ = "-=" if n.descending else "+="
                    host.append(pad + f"for (int {n.var} = {n.lo}; {n.var} {cmp} {n.hi}; "
                                f"{n.var} {op_} {n.step}) {{")
                    walk(n.body, scalars + [n.var], indent + 4)
                    host.append(pad + "}")
                else:
                    host.append(pad + launch([n], scalars, False))
            elif n.kind in ("assign", "decl"):
                host.append(pad + launch([n], scalars, False))
            else:
                raise Unsupported(f"host-level {n.kind}")

    walk(prog.roots, [], 8)
    copies_in, copies_out = [], []
    for ctype, name in prog.params:
        copies_in.append(f"        size_t n_{name} = extent_bytes({name}_vec, {row_bytes(prog, ctype, name)});\n"
                         f"        {ctype}* d_{name} = 0;\n"
                         f"        if (cudaMalloc(&d_{name}, n_{name} ? n_{name} : 16) != cudaSuccess) return 2;\n"
                         f"        cudaMemcpy(d_{name}, {name}_vec, n_{name}, cudaMemcpyHostToDevice);")
        copies_out.append(f"        cudaMemcpy({name}_vec, d_{name}, n_{name}, cudaMemcpyDeviceToHost);\n"
                          f"        cudaFree(d_{name});")
    alias_decl = "".join(f"        int {a} = 0;\n" for a in prog.alias_names)
    host_params = ", ".join(f"{c} *{n}_vec" for c, n in prog.params)
    nl = "\n"
    return f"""// generated by sf-cuda-cc: statement-for-statement CUDA translation
#include <cuda_runtime.h>
#include <malloc.h>
#include <math.h>
#include <stddef.h>

// the GridFunction buffers come from aligned_alloc (grid.cpp:58-64): the
// allocator's usable size bounds the array; round down to whole rows
static size_t extent_bytes(const void* p, size_t row) {{
    size_t n = malloc_usable_size(const_cast<void*>(p));
    return row ? n / row * row : n;
}}

// powf with a non-integral exponent (codegen.cpp:170-176): CUDA's double pow
// (<= 2 ulp) rounded once to float. glibc's powf (what the gcc build calls)
// is not always the correctly rounded result either, and double pow is left
// to CUDA's pow, so operators that use pow / powf are the one KNOWN
// non-bitwise case of this generic back end (the acoustic and diffusion hot
// paths have none; DESIGN.md section 9).
__device__ __forceinline__ float sf_powf(float a, float b) {{
    return (float)pow((double)a, (double)b);
}}
#define powf sf_powf

{nl.join(kernels)}

extern "C" int {prog.entry}({host_params}) {{
    {{
{nl.join(copies_in)}
{alias_decl}{nl.join(host)}
        if (cudaDeviceSynchronize() != cudaSuccess) return 3;
{nl.join(copies_out)}
    }}
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}}
"""


def row_bytes(prog: Program, ctype: str, name: str) -> int:
    size = {"float": 4, "double": 8, "int": 4}[ctype]
    dims = prog.arrays[name].dims
    n = size
    for d in dims:
        n *= d
    return n


# ---------------------------------------------------------------------------
# driver

def translate(src: str, generic: bool = False):
    """(kind, source_text, language) for the generated C translation unit."""
    prog = parse(src)
    op = None if generic else recognise(prog)
    if isinstance(op, AcousticOp):
        return "acoustic", emit_acoustic(op, prog.entry), "c++"
    if isinstance(op, DiffusionOp):
        return "diffusion", emit_diffusion(op, prog.entry), "c++"
    return "generic", emit_generic(prog), "cuda"


def build(src_path: str, out_path: str, generic: bool = False) -> str:
    with open(src_path) as f:
        src = f.read()
    kind, text, lang = translate(src, generic)
    lib_dir = HERE
    inc = os.path.join(ROOT, "include")
    with tempfile.TemporaryDirectory() as td:
        if lang == "c++":
            cpp = os.path.join(td, "op.cpp")
            with open(cpp, "w") as f:
                f.write(text)
            cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-I", inc, "-o", out_path, cpp,
                   "-L", lib_dir, "-lsf_b200", f"-Wl,-rpath,{lib_dir}"]
        else:
            cu = os.path.join(td, "op.cu")
            with open(cu, "w") as f:
                f.write(text)
            cmd = [NVCC, "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                   "--fmad=false", "-w", "-Xcompiler", "-fPIC", "-shared", "-ccbin", "g++", "-o",
                   out_path, cu]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise SystemExit(r.returncode)
    return kind


def main(argv=None, generic=False):
    """gcc-compatible command line: `... -o lib.so src.c [flags]` (jit.cpp:67-80)."""
    argv = list(sys.argv[1:] if argv is None else argv)
    out = None
    srcs = []
    i = 0
    while i < len(argv):
        a = argv[i]
        if a == "-o":
            out = argv[i + 1]
            i += 2
            continue
        if a.endswith(".c") or a.endswith(".cc"):
            srcs.append(a)
        i += 1
    if out is None or len(srcs) != 1:
        sys.stderr.write("sf-cuda-cc: need exactly one source and -o <lib>\n")
        return 2
    try:
        kind = build(srcs[0], out, generic or bool(os.environ.get("SF_CUDA_CC_GENERIC")))
    except Unsupported as e:
        sys.stderr.write(f"sf-cuda-cc: unsupported generated code: {e}\n")
        return 1
    if os.environ.get("SF_CUDA_CC_VERBOSE"):
        sys.stderr.write(f"sf-cuda-cc: {srcs[0]} -> {out} ({kind})\n")
    if os.environ.get("SF_CUDA_CC_LOG"):
        with open(os.environ["SF_CUDA_CC_LOG"], "a") as f:
            f.write(f"{kind} {out}\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
