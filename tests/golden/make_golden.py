"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in the build container (needs oracle/_ref/libsf_ref.so, i.e. the
reference compiled from /root/reference by `make -C oracle`):

    python tests/golden/make_golden.py

Outputs (committed):
  constants.json  folded fp32 constants and emitted term order of the
                  reference's generated stencil statements (parsed from
                  Operator::source(), codegen.cpp:411-502), acoustic 2D/3D,
                  orders 2-16, forward/adjoint, several (h, dt); diffusion
                  orders 2-16 with rational alpha/dx.
  fields.npz      small end-to-end runs of the reference's JIT kernel
                  (Operator::apply): final time slots and sparse traces.
  sparse.npz      interpolation_weights cells/weights for seeded points.
  medium.npz      build_medium m/eta for a small 3D model.
"""
from __future__ import annotations

import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import AcousticCase, Ref, ref_acoustic, ref_diffusion  # noqa: E402

ALIAS_RE = re.compile(r"^[uv]\[(t\d)\]((?:\[[^\]]+\])+)$")


def split_terms(rhs: str):
    """Top-level ' + ' / ' - ' split of an emitted expression."""
    terms, depth, cur, sign = [], 0, "", "+"
    i = 0
    if rhs.startswith("-"):
        sign, i = "-", 1
    while i < len(rhs):
        ch = rhs[i]
        if ch == "[" or ch == "(":
            depth += 1
        elif ch == "]" or ch == ")":
            depth -= 1
        if depth == 0 and rhs.startswith(" + ", i) or depth == 0 and rhs.startswith(" - ", i):
            terms.append((sign, cur))
            sign = rhs[i + 1]
            cur = ""
            i += 3
            continue
        cur += ch
        i += 1
    terms.append((sign, cur))
    return terms


def parse_float(lit: str) -> float:
    return float(np.float32(float(lit.rstrip("F"))))


def index_offsets(idx: str):
    """'[i1][i2 - 2][i3]' -> [0, -2, 0]"""
    out = []
    for part in re.findall(r"\[([^\]]+)\]", idx):
        mm = re.match(r"^i\d+(?: ([+-]) (\d+))?$", part.strip())
        assert mm, part
        out.append(0 if mm.group(1) is None else (int(mm.group(2)) * (1 if mm.group(1) == "+" else -1)))
    return out


def parse_acoustic(src: str, forward: bool):
    lines = [ln.strip() for ln in src.splitlines()]
    temps = {}
    stencil = None
    inject_scale = None
    for ln in lines:
        mm = re.match(r"^const float (temp\d) = (.*);$", ln)
        if mm:
            temps[mm.group(1)] = mm.group(2)
        if re.match(r"^[uv]\[t\d\]\[i1\]", ln) and "temp3" in ln:
            stencil = ln
        mm = re.match(r"^[uv]\[t\d\]\[\w+_ci\[p\]\[0\]\].* = ([0-9.e+-]+F)\*", ln)
        if mm and inject_scale is None:
            inject_scale = parse_float(mm.group(1))
    assert stencil is not None
    ce = parse_float(temps["temp0"].split("*")[0])
    assert temps["temp0"].split("*")[1].startswith("eta[")
    cm = parse_float(temps["temp1"].split("*")[0])
    assert temps["temp1"].split("*")[1].startswith("m[")
    assert temps["temp2"] == "temp0 + temp1" and temps["temp3"] == "1.0F/temp2"
    lhs, rhs = stencil.rstrip(";").split(" = ", 1)
    out_alias = ALIAS_RE.match(lhs).group(1)
    level = {("t0", True): "prev", ("t1", True): "cur", ("t2", False): "prev",
             ("t1", False): "cur"}
    terms = []
    for sign, body in split_terms(rhs):
        f = body.split("*")
        c = parse_float(f[0]) * (-1.0 if sign == "-" else 1.0)
        assert f[1] == "temp3", body
        rest = f[2:]
        if len(rest) == 2:  # time term: field * level
            fld = rest[0].split("[")[0]
            al = ALIAS_RE.match(rest[1])
            terms.append(["T", c, fld, level[(al.group(1), forward)]])
        else:
            al = ALIAS_RE.match(rest[0])
            assert level[(al.group(1), forward)] == "cur"
            offs = index_offsets(al.group(2))
            nz = [(a, o) for a, o in enumerate(offs) if o != 0]
            if not nz:
                terms.append(["C", c])
            else:
                assert len(nz) == 1
                terms.append(["N", c, nz[0][0], nz[0][1]])
    return {"ce": ce, "cm": cm, "out_alias": out_alias, "terms": terms,
            "inject_scale": inject_scale}


def parse_diffusion(src: str):
    stencil = [ln.strip() for ln in src.splitlines() if ln.strip().startswith("u[t1][i1][i2] =")]
    assert len(stencil) == 1
    rhs = stencil[0].rstrip(";").split(" = ", 1)[1]
    terms = []
    for sign, body in split_terms(rhs):
        f = body.split("*")
        if len(f) == 1:
            c, ref = 1.0, f[0]
        else:
            c, ref = parse_float(f[0]), f[1]
        c *= -1.0 if sign == "-" else 1.0
        al = ALIAS_RE.match(ref)
        offs = index_offsets(al.group(2))
        nz = [(a, o) for a, o in enumerate(offs) if o != 0]
        terms.append(["C", c] if not nz else ["N", c, nz[0][0], nz[0][1]])
    return {"terms": terms}


def main():
    ref = Ref()
    ref.set_threads(4)
    acoustic = []
    hdt = [(10.0, 1.6e-3), (15.0, 0.0), (12.5, 0.0), (10.0, 8.474e-4), (7.0, 1.0e-3)]
    for ndim in (2, 3):
        shape = (40, 36, 34)[:ndim] if ndim == 3 else (60, 52)
        for order in range(2, 17, 2):
            for forward in (True, False):
                for h, dt in hdt:
                    case = AcousticCase(shape=shape, nt=5, boundary_width=6, spacing=h, dt=0.0,
                                        space_order=order)
                    probe = ref_acoustic(ref, case, forward)
                    dt_use = dt if 0 < dt <= probe.dt else probe.dt
                    case.dt = dt_use
                    op = ref_acoustic(ref, case, forward)
                    d = parse_acoustic(op.source(), forward)
                    d.update({"ndim": ndim, "order": order, "forward": forward, "spacing": h,
                              "dt": dt_use})
                    acoustic.append(d)
    diffusion = []
    for order in range(2, 17, 2):
        for alpha, dx in [((1, 2), (1, 2047)), ((1, 1), (1, 1)), ((3, 7), (1, 49)),
                          ((1, 3), (2, 39))]:
            n = max(2 * order + 4, 20)
            op = ref_diffusion(ref, n, n, alpha, dx, 3, order)
            d = parse_diffusion(op.source())
            d.update({"order": order, "alpha": alpha, "dx": dx})
            diffusion.append(d)
    with open(os.path.join(HERE, "constants.json"), "w") as f:
        json.dump({"acoustic": acoustic, "diffusion": diffusion}, f, indent=0)

    fields = {}
    # the frozen golden kernel's own configuration (test_codegen.cpp:77-104)
    rng = np.random.default_rng(20161103)
    for tag, case, forward, random_residual in [
        ("golden3d_fwd", AcousticCase(shape=(24, 24, 20), nt=12, boundary_width=4), True, False),
        ("o8_3d_adj", AcousticCase(shape=(30, 28, 26), nt=15, boundary_width=5, spacing=10.0,
                                   space_order=8), False, True),
        ("o4_2d_fwd", AcousticCase(shape=(40, 36), nt=30, boundary_width=6, space_order=4), True,
         False),
    ]:
        op = ref_acoustic(ref, case, forward)
        nd = len(case.shape)
        nsrc = 1
        nrec = 8
        if random_residual:
            res = rng.standard_normal((case.nt, nrec)).astype(np.float32)
            op.set("rec", res)
            fields[tag + "_residual"] = res
        op.apply()
        fname = "u" if forward else "v"
        fields[tag + "_field"] = op.get(fname, np.float32, (3,) + tuple(case.shape))
        fields[tag + "_src"] = op.get("src", np.float32, (case.nt, nsrc))
        fields[tag + "_rec"] = op.get("rec", np.float32, (case.nt, nrec))
        fields[tag + "_src_ci"] = op.get("src_ci", np.int32, (nsrc, nd))
        fields[tag + "_src_w"] = op.get("src_w", np.float32, (nsrc, 1 << nd))
        fields[tag + "_rec_ci"] = op.get("rec_ci", np.int32, (nrec, nd))
        fields[tag + "_rec_w"] = op.get("rec_w", np.float32, (nrec, 1 << nd))
        fields[tag + "_m"] = op.get("m", np.float32, tuple(case.shape))
        fields[tag + "_eta"] = op.get("eta", np.float32, tuple(case.shape))
        fields[tag + "_meta"] = np.array([case.nt, case.space_order, int(forward), op.dt,
                                          case.spacing], np.float64)
    for tag, n, nt, order, alpha, dx in [("diff_o2", 64, 30, 2, (1, 2), (1, 63)),
                                         ("diff_o4", 33, 7, 4, (1, 1), (1, 1))]:
        op = ref_diffusion(ref, n, n, alpha, dx, nt, order)
        u0 = np.zeros((n, n), np.float32)
        u0[1:-1, 1:-1] = rng.random((n - 2, n - 2)).astype(np.float32)
        op.set("u", np.stack([u0, u0]))
        op.apply()
        fields[tag + "_u0"] = u0
        fields[tag + "_out"] = op.get("u", np.float32, (2, n, n))
        fields[tag + "_meta"] = np.array([n, nt, order, alpha[0], alpha[1], dx[0], dx[1]],
                                         np.int64)
    np.savez_compressed(os.path.join(HERE, "fields.npz"), **fields)

    # interpolation weights (criterion-10-like seeded points + node/centre)
    pts = np.concatenate([rng.uniform(0.5, 18.0, (100, 3)),
                          np.array([[2.0, 3.0, 4.0], [2.5, 3.5, 4.5], [0.0, 0.0, 0.0],
                                    [18.0, 18.0, 18.0]])])
    cells = np.zeros((len(pts), 3), np.int64)
    wts = np.zeros((len(pts), 8), np.float64)
    ext = np.array([20, 20, 20], np.int64)
    import ctypes as C
    for i, p in enumerate(pts):
        cell = (C.c_long * 3)()
        w = np.zeros(8, np.float64)
        assert ref.lib.sfref_interp_weights(3, np.ascontiguousarray(p), 1.0, ext, cell, w) == 0
        cells[i] = list(cell)
        wts[i] = w
    np.savez_compressed(os.path.join(HERE, "sparse.npz"), coords=pts, cells=cells,
                        weights=wts, extents=ext)

    case = AcousticCase(shape=(30, 28, 26), nt=1, boundary_width=6, spacing=12.5,
                        v_top=1700.0, v_bottom=3100.0)
    op = ref_acoustic(ref, case, True)
    np.savez_compressed(os.path.join(HERE, "medium.npz"),
                        m=op.get("m", np.float32, case.shape),
                        eta=op.get("eta", np.float32, case.shape),
                        meta=np.array([30, 28, 26, 6, 12.5, 1700.0, 3100.0]))
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
