"""Host-side logic of the product library (no GPU needed): the C ABI loads
and exports every declared symbol, the folded constants match the
reference's generated source, and the setup mirrors (interpolation weights,
medium, stability bound, Ricker, RNG) match the reference bit for bit."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, gpu_available


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def header_symbols():
    with open(os.path.join(ROOT, "include", "sf_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_1609_03361_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(_lib.EXPORTS) == syms
    lib = C.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    from paper_1609_03361_b200 import _lib
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(gpu_available(), reason="checks the no-device failure mode")
def test_no_cpu_fallback_without_device():
    import paper_1609_03361_b200 as sf
    with pytest.raises(sf.CudaError):
        sf.acoustic_build(sf.AcousticModel(shape=(24, 24, 20), nt=2, boundary_width=4), True)
    with pytest.raises(sf.CudaError):
        sf.make_diffusion_operator(sf.DiffusionConfig(nx=16, ny=16, nt=1))


def product_terms(ndim, order, forward, dt, h):
    from paper_1609_03361_b200._lib import lib
    out = np.zeros(15, np.float32)
    sel = np.zeros(3, np.int32)
    assert lib.sf_acoustic_constants(ndim, order, int(forward), dt, h, out, sel) == 0
    r = order // 2
    terms = []
    for k in range(3):
        terms.append(["T", float(out[2 + k]), "m" if sel[k] // 2 else "eta",
                      "cur" if sel[k] % 2 else "prev"])
    terms.append(["C", float(out[5])])
    for axis in reversed(range(ndim)):
        for j in list(range(-r, 0)) + list(range(1, r + 1)):
            terms.append(["N", float(out[6 + abs(j) - 1]), axis, j])
    return out, terms


def same_terms(a, b):
    return len(a) == len(b) and all(
        x[0] == y[0] and np.float32(x[1]).view(np.uint32) == np.float32(y[1]).view(np.uint32)
        and x[2:] == y[2:] for x, y in zip(a, b))


def test_product_constants_match_reference_source(golden):
    cases = golden["constants"]["acoustic"]
    assert len(cases) == 160
    for case in cases:
        out, terms = product_terms(case["ndim"], case["order"], case["forward"], case["dt"],
                                   case["spacing"])
        assert np.float32(out[0]) == np.float32(case["ce"])
        assert np.float32(out[1]) == np.float32(case["cm"])
        assert np.float32(out[14]) == np.float32(case["inject_scale"])
        assert same_terms(terms, case["terms"]), (case["ndim"], case["order"], case["forward"])


def test_product_diffusion_constants(golden):
    from paper_1609_03361_b200._lib import lib
    for case in golden["constants"]["diffusion"]:
        c0 = C.c_float()
        has = C.c_int()
        cj = np.zeros(8, np.float32)
        (an, ad), (dn, dd) = case["alpha"], case["dx"]
        assert lib.sf_diffusion_constants(case["order"], an, ad, dn, dd, C.byref(c0),
                                          C.byref(has), cj) == 0
        r = case["order"] // 2
        terms = [["C", c0.value]] if has.value else []
        for axis in (1, 0):
            for j in list(range(-r, 0)) + list(range(1, r + 1)):
                terms.append(["N", float(cj[abs(j) - 1]), axis, j])
        assert same_terms(terms, case["terms"]), case


def test_interpolation_weights_bit_exact(golden):
    import paper_1609_03361_b200 as sf
    s = golden["sparse"]
    for p, c in enumerate(s["coords"]):
        cell, w = sf.interpolation_weights(c, 1.0, s["extents"])
        assert np.array_equal(cell.astype(np.int64), s["cells"][p])
        assert np.array_equal(bits(w), bits(s["weights"][p].astype(np.float32)))
        assert abs(float(w.astype(np.float64).sum()) - 1.0) <= 1e-6  # partition of unity


def test_interpolation_out_of_domain():
    import paper_1609_03361_b200 as sf
    # test_sparse.cpp:64-72: below the origin / beyond the last cell
    with pytest.raises(sf.OutOfDomainError):
        sf.interpolation_weights([-0.1, 1.0], 1.0, [10, 10])
    with pytest.raises(sf.OutOfDomainError):
        sf.interpolation_weights([9.0, 1.0], 1.0, [10, 10])
    cell, w = sf.interpolation_weights([8.999, 1.0], 1.0, [10, 10])
    assert list(cell) == [8, 1]
    # on a node: all weight on corner 0; at a centre: equal weights
    cell, w = sf.interpolation_weights([3.0, 4.0, 5.0], 1.0, [10, 10, 10])
    assert list(cell) == [3, 4, 5] and w[0] == 1.0 and not w[1:].any()
    cell, w = sf.interpolation_weights([3.5, 4.5, 5.5], 1.0, [10, 10, 10])
    assert np.all(w == np.float32(0.125))


def test_medium_bit_exact(golden):
    import paper_1609_03361_b200 as sf
    md = golden["medium"]
    n0, n1, n2, bw, h, vt, vb = md["meta"]
    model = sf.AcousticModel(shape=(int(n0), int(n1), int(n2)), boundary_width=int(bw),
                             spacing=float(h), v_top=float(vt), v_bottom=float(vb))
    g = sf.Grid()
    m, eta = sf.build_medium(g, model)
    assert np.array_equal(bits(m.data), bits(md["m"]))
    assert np.array_equal(bits(eta.data), bits(md["eta"]))


def test_stable_dt_ricker_rng_vs_reference(ref, port):
    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200.api import _mt19937_64_uniform
    for ndim in (2, 3):
        for order in range(2, 17, 2):
            shape = np.array([40] * ndim, np.int64)
            want = ref.lib.sfref_acoustic_stable_dt(ndim, shape, 12.5, order, 1500.0, 4500.0)
            m = sf.AcousticModel(shape=(40,) * ndim, spacing=12.5, space_order=order,
                                 v_top=1500.0, v_bottom=4500.0)
            assert m.stable_dt() == want
    for t in np.linspace(0, 0.3, 37):
        assert sf.ricker_wavelet(10.0, t, 0.1) == ref.lib.sfref_ricker(10.0, t, 0.1)
    ref.lib.sfref_mt_uniform.argtypes = [C.c_uint, C.c_long, C.c_double, C.c_double,
                                         np.ctypeslib.ndpointer(np.float64)]
    want = np.zeros(500, np.float64)
    ref.lib.sfref_mt_uniform(7, 500, -1.0, 1.0, want)
    assert np.array_equal(_mt19937_64_uniform(7, 500, -1.0, 1.0), want)


def test_cfl_guard():
    import paper_1609_03361_b200 as sf
    # test_apps.cpp:210-216
    m = sf.AcousticModel(shape=(40, 40), nt=10)
    m.dt = m.stable_dt() * 2.0
    with pytest.raises(sf.CflViolationError):
        sf.acoustic_forward(m)


def test_invalid_orders_and_shapes():
    import paper_1609_03361_b200 as sf
    with pytest.raises(sf.InvalidOrderError):
        sf.Grid().create_dense("m", (10, 10), 3)
    with pytest.raises(sf.InvalidShapeError):
        sf.Grid().create_dense("m", (4, 10), 4)


def test_reference_arm_line_on_cpu():
    """bench.py --impl reference (the driver's reference arm) runs the
    reference's own CPU path and prints the contract's JSON line; C1 is the
    reference's CPU-runnable case and takes a second here."""
    import json
    import subprocess
    import sys
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsf_ref.so")):
        pytest.skip("reference not built (oracle/_ref)")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GPts/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "GPts/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("c1: 2D diffusion 2048^2")
    assert line["ms_per_step"] > 0 and line["higher_is_better"] is True


def test_reference_arm_never_loads_the_product():
    """The reference arm builds its case through oracle/ alone: after a full
    `bench.py --impl reference` run the process has neither imported this
    package nor mapped libsf_b200.so (the driver checks the mapped .so files)."""
    import subprocess
    import sys
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsf_ref.so")):
        pytest.skip("reference not built (oracle/_ref)")
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', "
            "'--steps', '1', '--warmup', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "sys.stderr.write('PRODUCT' if ('paper_1609_03361_b200' in sys.modules "
            "or 'libsf_b200' in maps) else 'CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, check=True)
    assert r.stderr.strip().endswith("CLEAN"), r.stderr[-500:]
