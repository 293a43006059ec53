"""Pin the C restatement (oracle/sf_port.c) before trusting it as the checker.

Against: the committed golden fixtures produced by the reference itself
(tests/golden/make_golden.py), and — when oracle/_ref/libsf_ref.so is built —
the live reference on fresh seeded inputs. CPU only.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle_lib import AcousticCase, ref_acoustic, ref_diffusion


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def port_terms(c):
    """Expand the port's constants to the emitted term list."""
    r = c.order // 2
    terms = []
    for k in range(3):
        terms.append(["T", c.tc[k], "m" if c.tfield[k] else "eta", "cur" if c.tlevel[k] else "prev"])
    terms.append(["C", c.c0])
    for axis in reversed(range(c.ndim)):
        for j in list(range(-r, 0)) + list(range(1, r + 1)):
            terms.append(["N", c.cj[abs(j) - 1], axis, j])
    return terms


def same_terms(a, b):
    if len(a) != len(b):
        return False
    for x, y in zip(a, b):
        if x[0] != y[0] or np.float32(x[1]).view(np.uint32) != np.float32(y[1]).view(np.uint32):
            return False
        if x[2:] != y[2:]:
            return False
    return True


def test_fd_weights_known_values(port):
    # fd.cpp reference values (test_fd.cpp: [-1/12, 4/3, -5/2, 4/3, -1/12])
    w = [Fraction(n, d) for n, d in port.fd_weights2(4)]
    assert w == [Fraction(-1, 12), Fraction(4, 3), Fraction(-5, 2), Fraction(4, 3),
                 Fraction(-1, 12)]
    from paper_1609_03361_b200.fd import fd_weights2
    for order in range(2, 17, 2):
        assert [Fraction(n, d) for n, d in port.fd_weights2(order)] == fd_weights2(order)
        assert sum(fd_weights2(order)) == 0


def test_port_constants_match_reference_source(port, golden):
    for case in golden["constants"]["acoustic"]:
        c = port.coefs(case["ndim"], case["order"], case["forward"], case["dt"], case["spacing"])
        assert np.float32(c.ce) == np.float32(case["ce"])
        assert np.float32(c.cm) == np.float32(case["cm"])
        assert np.float32(c.src_scale) == np.float32(case["inject_scale"])
        assert same_terms(port_terms(c), case["terms"]), case


def test_port_diffusion_constants(port, golden):
    for case in golden["constants"]["diffusion"]:
        c0, has, cj = port.diffusion_coefs(tuple(case["alpha"]), tuple(case["dx"]), case["order"])
        r = case["order"] // 2
        terms = [["C", c0]] if has else []
        for axis in (1, 0):
            for j in list(range(-r, 0)) + list(range(1, r + 1)):
                terms.append(["N", cj[abs(j) - 1], axis, j])
        assert same_terms(terms, case["terms"]), case


def _golden_acoustic(port, f, tag):
    nt, order, forward, dt, h = f[tag + "_meta"]
    nt, order, forward = int(nt), int(order), bool(forward)
    shape = f[tag + "_m"].shape
    c = port.coefs(len(shape), order, forward, dt, h)
    u = np.zeros((3,) + shape, np.float32)
    src = f[tag + "_src"].copy() if forward else np.zeros_like(f[tag + "_src"])
    rec = np.zeros_like(f[tag + "_rec"]) if forward else f[tag + "_residual"].copy()
    args = (f[tag + "_m"], f[tag + "_eta"])
    if forward:
        port.acoustic_run(c, u, *args, src, f[tag + "_src_ci"], f[tag + "_src_w"], rec,
                          f[tag + "_rec_ci"], f[tag + "_rec_w"], nt)
        return u, rec
    port.acoustic_run(c, u, *args, rec, f[tag + "_rec_ci"], f[tag + "_rec_w"], src,
                      f[tag + "_src_ci"], f[tag + "_src_w"], nt)
    return u, src


@pytest.mark.parametrize("tag", ["golden3d_fwd", "o8_3d_adj", "o4_2d_fwd"])
def test_port_reproduces_reference_fields(port, golden, tag):
    f = golden["fields"]
    u, traces = _golden_acoustic(port, f, tag)
    assert np.array_equal(bits(u), bits(f[tag + "_field"]))
    forward = bool(f[tag + "_meta"][2])
    want = f[tag + "_rec"] if forward else f[tag + "_src"]
    assert np.array_equal(bits(traces), bits(want))
    assert np.abs(u).max() > 0


@pytest.mark.parametrize("tag", ["diff_o2", "diff_o4"])
def test_port_reproduces_reference_diffusion(port, golden, tag):
    f = golden["fields"]
    n, nt, order, an, ad, dn, dd = (int(x) for x in f[tag + "_meta"])
    u = np.stack([f[tag + "_u0"], f[tag + "_u0"]]).astype(np.float32)
    port.diffusion_run(u, order, (an, ad), (dn, dd), nt)
    assert np.array_equal(bits(u), bits(f[tag + "_out"]))


def test_port_interpolation_and_medium(port, golden):
    s = golden["sparse"]
    ci, w = port.interp(s["coords"], 1.0, s["extents"])
    assert np.array_equal(ci.astype(np.int64), s["cells"])
    assert np.array_equal(bits(w), bits(s["weights"].astype(np.float32)))
    md = golden["medium"]
    n0, n1, n2, bw, h, vt, vb = md["meta"]
    m, eta = port.medium((int(n0), int(n1), int(n2)), int(bw), h, vt, vb)
    assert np.array_equal(bits(m), bits(md["m"]))
    assert np.array_equal(bits(eta), bits(md["eta"]))


# -- live reference (when built) ------------------------------------------

@pytest.mark.parametrize("order,forward", [(2, True), (6, False), (12, True), (16, False)])
def test_port_vs_live_reference_random_medium(port, ref, order, forward):
    rng = np.random.default_rng(order)
    shape = (26, 24, 22)
    case = AcousticCase(shape=shape, nt=10, boundary_width=4, spacing=10.0, space_order=order,
                        v_top=4500.0, v_bottom=4500.0)
    op = ref_acoustic(ref, case, forward)
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 4, 10.0, 1500.0)
    op.set("m", m)
    op.set("eta", eta)
    nrec = 8
    src_ci = op.get("src_ci", np.int32, (1, 3))
    src_w = op.get("src_w", np.float32, (1, 8))
    rec_ci = op.get("rec_ci", np.int32, (nrec, 3))
    rec_w = op.get("rec_w", np.float32, (nrec, 8))
    c = port.coefs(3, order, forward, op.dt, 10.0)
    u = np.zeros((3,) + shape, np.float32)
    if forward:
        src = op.get("src", np.float32, (10, 1))
        rec = np.zeros((10, nrec), np.float32)
        op.apply()
        port.acoustic_run(c, u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w, 10)
        got, want = rec, op.get("rec", np.float32, (10, nrec))
    else:
        rec = rng.standard_normal((10, nrec)).astype(np.float32)
        op.set("rec", rec)
        src = np.zeros((10, 1), np.float32)
        op.apply()
        port.acoustic_run(c, u, m, eta, rec, rec_ci, rec_w, src, src_ci, src_w, 10)
        got, want = src, op.get("src", np.float32, (10, 1))
    assert np.array_equal(bits(u), bits(op.get("u" if forward else "v", np.float32, (3,) + shape)))
    assert np.array_equal(bits(got), bits(want))


def test_port_vs_live_reference_diffusion(port, ref):
    rng = np.random.default_rng(3)
    for n, nt, order, alpha, dx in [(40, 9, 2, (1, 2), (1, 39)), (30, 5, 8, (2, 3), (1, 29))]:
        op = ref_diffusion(ref, n, n, alpha, dx, nt, order)
        u0 = np.zeros((n, n), np.float32)
        u0[1:-1, 1:-1] = rng.random((n - 2, n - 2))
        op.set("u", np.stack([u0, u0]))
        op.apply()
        u = np.stack([u0, u0])
        port.diffusion_run(u, order, alpha, dx, nt)
        assert np.array_equal(bits(u), bits(op.get("u", np.float32, (2, n, n))))
