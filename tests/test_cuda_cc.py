"""sf-cuda-cc: the reference's own Operator pipeline compiled onto the B200.

The reference JIT-compiles every operator through $STENCILFORGE_CC
(jit.cpp:84-95). These tests build operators with the unmodified reference
(oracle/_ref/libsf_ref.so), once with its default gcc toolchain and once with
STENCILFORGE_CC=bin/sf-cuda-cc, and require the two runs to leave bitwise
identical buffers. The CPU tests check the source front end: every lifted
literal equals the library's own folded constant, and both back ends build.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle_lib import AcousticCase, have_ref, ref_acoustic, ref_diffusion

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "bin", "sf-cuda-cc")

needs_ref = pytest.mark.skipif(not have_ref(), reason="reference not built (oracle/_ref)")

ACOUSTIC = [(shape, order, fwd)
            for shape in ((40, 36), (26, 24, 22))
            for order in (2, 4, 8, 16)
            for fwd in (True, False)]
DIFFUSION = [2, 4, 8, 16]


def _case(shape, order, nt=9):
    ndim = len(shape)
    return AcousticCase(shape=shape, boundary_width=4, nt=nt, spacing=12.0, space_order=order,
                        src_coords=[[130.0 + 3 * k] * ndim for k in range(2)],
                        rec_coords=[[40.0 + 17.5 * i, 200.0 - 9 * i, 55.0][:ndim]
                                    for i in range(5)])


def _buffers(op, names):
    out = {}
    for name in names:
        n = op.ref.lib.sfref_buffer_bytes(op.h, name.encode())
        dt = np.int32 if name.endswith("_ci") else np.float32
        out[name] = op.get(name, dt, (n // 4,))
    return out


ACOUSTIC_ARGS = ["m", "eta", "src", "src_ci", "src_w", "rec", "rec_ci", "rec_w"]


@needs_ref
@pytest.mark.parametrize("shape,order,fwd", ACOUSTIC)
def test_lifted_acoustic_constants_match_library(ref, shape, order, fwd):
    from paper_1609_03361_b200 import cuda_cc
    from paper_1609_03361_b200._lib import lib
    op = ref_acoustic(ref, _case(shape, order), fwd)
    prog = cuda_cc.parse(op.source())
    got = cuda_cc.recognise(prog)
    assert isinstance(got, cuda_cc.AcousticOp)
    assert got.shape == tuple(shape) and got.order == order and got.forward == fwd
    assert (got.n_src, got.n_rec, got.nt) == (2, 5, 9)
    want = np.zeros(15, np.float32)
    sel = np.zeros(3, np.int32)
    assert lib.sf_acoustic_constants(len(shape), order, int(fwd), op.dt, 12.0,
                                     want, sel) == 0
    assert np.array_equal(np.asarray(got.constants, np.float32).view(np.uint32),
                          want.view(np.uint32))
    assert list(sel) == got.tsel


@needs_ref
@pytest.mark.parametrize("order", DIFFUSION)
def test_lifted_diffusion_constants_match_library(ref, order):
    from paper_1609_03361_b200 import cuda_cc
    from paper_1609_03361_b200._lib import lib
    op = ref_diffusion(ref, 50, 40, (1, 2), (1, 10), 5, order)
    got = cuda_cc.recognise(cuda_cc.parse(op.source()))
    assert isinstance(got, cuda_cc.DiffusionOp)
    c0, has = C.c_float(), C.c_int()
    cj = np.zeros(8, np.float32)
    assert lib.sf_diffusion_constants(order, 1, 2, 1, 10, C.byref(c0), C.byref(has),
                                      cj) == 0
    assert bool(has.value) == got.has_c0
    if got.has_c0:
        assert np.float32(c0.value) == np.float32(got.c0)
    assert np.array_equal(np.asarray(got.cj, np.float32), cj)


BLOCKINGS = [(8, 0, 16), (4, 4, 4), (0, 3, 0)]


@needs_ref
@pytest.mark.parametrize("blocking", BLOCKINGS)
def test_blocked_sources_are_unblocked(ref, blocking):
    """AcousticModel/DiffusionConfig::blocking (opt.cpp:136-200) wraps the
    nest in block loops with capped inner bounds; the front end restores the
    plain nest and still recognises the operator with the same constants."""
    from paper_1609_03361_b200 import cuda_cc
    plain = cuda_cc.recognise(cuda_cc.parse(ref_acoustic(ref, _case((26, 24, 22), 4), True)
                                            .source()))
    ref.set_blocking(blocking)
    try:
        src = ref_acoustic(ref, _case((26, 24, 22), 4), True).source()
        dsrc = ref_diffusion(ref, 50, 40, (1, 2), (1, 10), 5, 4).source()
    finally:
        ref.set_blocking()
    assert "_hi = " in src
    assert cuda_cc.recognise(cuda_cc.parse(src)) == plain
    assert isinstance(cuda_cc.recognise(cuda_cc.parse(dsrc)), cuda_cc.DiffusionOp)


def test_unrecognised_source_falls_back_to_generic():
    from paper_1609_03361_b200 import cuda_cc
    src = """#include <math.h>

int Operator(float *a_vec, float *b_vec)
{
  float (*a)[10] = (float (*)[10]) a_vec;
  float *b = b_vec;
  {
    #pragma omp parallel
    {
      #pragma omp for schedule(static)
      for (int i1 = 0; i1 < 6; i1 += 1)
      {
        #pragma omp simd aligned(a:64)
        for (int i2 = 1; i2 < 9; i2 += 1)
        {
          a[i1][i2] = 5.0e-1F*a[i1][i2 - 1] + b[i2];
        }
      }
    }
  }
  return 0;
}
"""
    kind, text, lang = cuda_cc.translate(src)
    assert kind == "generic" and lang == "cuda"
    assert "__global__ void sfk0" in text and "a[i1][i2] = 5.0e-1F*a[i1][i2 - 1] + b[i2];" in text


# an operator outside the recognised families, in the reference's emitted
# form (codegen.cpp:411-502): an f64 "save every level" time loop without an
# alias block, an in-place recurrence, a 1-D nest with powf, a descending loop
CUSTOM = """#include <math.h>

int Operator(double *a_vec, float *b_vec, float *c_vec)
{
  double (*a)[40][30] = (double (*)[40][30]) a_vec;
  float (*b)[33] = (float (*)[33]) b_vec;
  float *c = c_vec;
  {
    for (int i3 = 0; i3 < 6; i3 += 1)
    {
      for (int i1 = 1; i1 < 39; i1 += 1)
      {
        for (int i2 = 1; i2 < 29; i2 += 1)
        {
          a[i3 + 1][i1][i2] = 2.5e-1*a[i3][i1 - 1][i2] + 2.5e-1*a[i3][i1 + 1][i2] + 2.5e-1*a[i3][i1][i2 - 1] + 2.5e-1*a[i3][i1][i2 + 1] - 1.0e-3*a[i3 + 1][i1][i2];
        }
      }
      for (int i1 = 1; i1 < 33; i1 += 1)
      {
        b[i3][i1] = 5.0e-1F*b[i3][i1 - 1] + c[i1];
      }
      for (int i1 = 0; i1 < 33; i1 += 1)
      {
        const float temp0 = powf(c[i1], 1.5e0F);
        c[i1] = temp0/(1.0F + c[i1]);
      }
    }
    for (int i1 = 31; i1 >= 1; i1 -= 1)
    {
      b[6][i1] = b[6][i1 + 1] - 2.5e-1F*b[5][i1];
    }
  }
  return 0;
}
"""
CUSTOM_SHAPES = [("a", np.float64, (7, 40, 30)), ("b", np.float32, (7, 33)),
                 ("c", np.float32, (33,))]


def test_generic_schedule_decisions():
    """Parallel only where the dependence test proves it; recurrences and
    indirect (colliding) writes stay sequential, in order."""
    from paper_1609_03361_b200 import cuda_cc
    prog = cuda_cc.parse(CUSTOM)
    text = cuda_cc.emit_generic(prog)
    host = text[text.index('extern "C"'):]
    launches = [ln.strip() for ln in host.splitlines() if "<<<" in ln]
    # a-nest: parallel 2-D; b recurrence: one thread; c: parallel 1-D;
    # descending recurrence: one thread
    assert ["<<<1, 1>>>" in ln for ln in launches] == [False, True, False, True]
    assert "for (int i3 = 0; i3 < 6; i3 += 1) {" in host


@needs_ref
def test_generic_schedule_of_acoustic(ref):
    from paper_1609_03361_b200 import cuda_cc
    src = ref_acoustic(ref, _case((26, 24, 22), 4), True).source()
    text = cuda_cc.emit_generic(cuda_cc.parse(src))
    launches = [ln for ln in text[text.index('extern "C"'):].splitlines() if "<<<" in ln]
    assert ["<<<1, 1>>>" in ln for ln in launches] == [False, True, False]


@needs_ref
@pytest.mark.parametrize("generic", [False, True])
def test_tool_builds_shared_library(ref, tmp_path, generic):
    op = ref_acoustic(ref, _case((26, 24, 22), 8), True)
    src = tmp_path / "kernel.c"
    src.write_text(op.source())
    lib = tmp_path / "kernel.so"
    env = dict(os.environ, SF_CUDA_CC_LOG=str(tmp_path / "log"))
    # the exact command line jit.cpp:67-80 issues
    cmd = [TOOL + ("-generic" if generic else ""), "-std=c99", "-O3", "-march=native", "-fPIC", "-shared", "-ffp-contract=off",
           "-fopenmp", "-o", str(lib), str(src), "-lm"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    syms = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True,
                          text=True).stdout
    assert " T Operator" in syms
    assert (tmp_path / "log").read_text().split()[0] == ("generic" if generic else "acoustic")


def test_tool_rejects_bad_command_line(tmp_path):
    r = subprocess.run([TOOL, "-O3"], capture_output=True, text=True)
    assert r.returncode == 2


# ---------------------------------------------------------------------------
# the reference's pipeline end to end on the GPU


@pytest.fixture(scope="module")
def sf():
    import paper_1609_03361_b200 as sf
    if sf._lib.lib.sf_device_count() < 1:
        pytest.fail("no CUDA device: the GPU tests need a B200")
    return sf


@pytest.fixture
def cuda_cc_env(monkeypatch, tmp_path):
    """Point the reference at sf-cuda-cc (the generic flavour is a separate
    executable so the reference's JIT cache, keyed on the executable, keeps
    the two builds apart) and return the tool's build log."""
    log = tmp_path / "sf-cuda-cc.log"

    def use(generic):
        monkeypatch.setenv("STENCILFORGE_CC", TOOL + ("-generic" if generic else ""))
        monkeypatch.setenv("SF_CUDA_CC_LOG", str(log))
        return log
    return use


def _run_acoustic(ref, shape, order, fwd, seed, blocking=()):
    ref.set_blocking(blocking)
    try:
        op = ref_acoustic(ref, _case(shape, order), fwd)
    finally:
        ref.set_blocking()
    rng = np.random.default_rng(seed)
    field = "u" if fwd else "v"
    if not fwd:
        rec = _buffers(op, ["rec"])["rec"]
        op.set("rec", rng.standard_normal(rec.shape).astype(np.float32))
    # a non-zero start state exercises every slot of the time buffer
    n = op.ref.lib.sfref_buffer_bytes(op.h, field.encode()) // 4
    op.set(field, (1e-3 * rng.standard_normal(n)).astype(np.float32))
    op.apply()
    return _buffers(op, [field] + ACOUSTIC_ARGS)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("shape,order,fwd", ACOUSTIC)
def test_reference_pipeline_on_gpu_acoustic(sf, ref, cuda_cc_env, shape, order, fwd, generic):
    want = _run_acoustic(ref, shape, order, fwd, 7)          # reference, gcc
    log = cuda_cc_env(generic)
    got = _run_acoustic(ref, shape, order, fwd, 7)           # reference, sf-cuda-cc
    assert log.read_text().split()[0] == ("generic" if generic else "acoustic")
    for name in want:
        assert np.array_equal(got[name].view(np.uint32), want[name].view(np.uint32)), name


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("blocking", BLOCKINGS)
def test_reference_pipeline_on_gpu_blocked(sf, ref, cuda_cc_env, blocking, generic):
    want = _run_acoustic(ref, (26, 24, 22), 4, False, 3, blocking)
    log = cuda_cc_env(generic)
    got = _run_acoustic(ref, (26, 24, 22), 4, False, 3, blocking)
    assert log.read_text().split()[0] == ("generic" if generic else "acoustic")
    for name in want:
        assert np.array_equal(got[name].view(np.uint32), want[name].view(np.uint32)), name


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("order", DIFFUSION)
def test_reference_pipeline_on_gpu_diffusion(sf, ref, cuda_cc_env, order, generic):
    def run():
        op = ref_diffusion(ref, 70, 66, (1, 2), (1, 10), 23, order)
        rng = np.random.default_rng(order)
        op.set("u", rng.random(2 * 70 * 66).astype(np.float32))
        op.apply()
        return op.get("u", np.float32, (2, 70, 66))
    want = run()
    log = cuda_cc_env(generic)
    got = run()
    assert log.read_text().split()[0] == ("generic" if generic else "diffusion")
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def _aligned_buffers(arrays):
    """Host buffers from aligned_alloc, as GridFunction allocates them
    (grid.cpp:58-64), so the generic translation can size them."""
    libc = C.CDLL(None)
    libc.aligned_alloc.restype = C.c_void_p
    libc.aligned_alloc.argtypes = [C.c_size_t, C.c_size_t]
    libc.free.argtypes = [C.c_void_p]
    bufs = []
    for arr in arrays:
        nbytes = (arr.nbytes + 63) // 64 * 64
        p = libc.aligned_alloc(64, nbytes)
        C.memmove(p, arr.ctypes.data, arr.nbytes)
        bufs.append(p)
    return libc, bufs


@pytest.mark.gpu
def test_generic_translation_matches_gcc(sf, tmp_path):
    """The custom operator built by gcc (the reference's default toolchain
    flags, jit.cpp:70) and by sf-cuda-cc leave bitwise-identical buffers."""
    src = tmp_path / "custom.c"
    src.write_text(CUSTOM)
    gcc_lib, cc_lib = tmp_path / "gcc.so", tmp_path / "cc.so"
    subprocess.run(["gcc", "-std=c99", "-O3", "-march=native", "-fPIC", "-shared",
                    "-ffp-contract=off", "-o", str(gcc_lib), str(src), "-lm"], check=True)
    r = subprocess.run([TOOL, "-std=c99", "-O3", "-fPIC", "-shared", "-o", str(cc_lib), str(src),
                        "-lm"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rng = np.random.default_rng(11)
    init = [rng.random(shape).astype(dt) for _, dt, shape in CUSTOM_SHAPES]
    results = []
    for lib_path in (gcc_lib, cc_lib):
        lib = C.CDLL(str(lib_path))
        libc, bufs = _aligned_buffers(init)
        assert lib.Operator(*[C.c_void_p(b) for b in bufs]) == 0
        out = []
        for b, arr in zip(bufs, init):
            got = np.empty_like(arr)
            C.memmove(got.ctypes.data, b, arr.nbytes)
            out.append(got)
            libc.free(b)
        results.append(out)
    for (name, _, _), want, got in zip(CUSTOM_SHAPES, *results):
        assert np.array_equal(want.view(np.uint8), got.view(np.uint8)), name


GOLDEN_DIR = "/root/reference/proj/tests/golden"


@pytest.mark.skipif(not os.path.isdir(GOLDEN_DIR), reason="reference golden sources absent")
def test_reference_golden_sources_are_recognised():
    """The reference's own golden generated kernels (test_codegen.cpp:77-104,
    acceptance.cpp:139-166) go through the front end as the operators they
    are, with the literals the library folds for those configurations."""
    from paper_1609_03361_b200 import cuda_cc
    from paper_1609_03361_b200._lib import lib
    with open(os.path.join(GOLDEN_DIR, "diffusion_1000.c")) as f:
        d = cuda_cc.recognise(cuda_cc.parse(f.read()))
    assert isinstance(d, cuda_cc.DiffusionOp)
    assert d.shape == (1000, 1000) and d.nt == 500 and d.order == 2 and not d.has_c0
    assert np.float32(d.cj[0]) == np.float32(0.25)
    with open(os.path.join(GOLDEN_DIR, "acoustic_3d.c")) as f:
        a = cuda_cc.recognise(cuda_cc.parse(f.read()))
    assert isinstance(a, cuda_cc.AcousticOp)
    assert a.forward and a.shape == (24, 24, 20) and a.order == 2 and a.nt == 12
    assert a.tsel == [0, 2, 3]
    # every lifted literal is a float the library produces for some dt: the
    # golden file's ce/cm pair pins dt, the rest must then agree bitwise
    ce, cm = a.constants[0], a.constants[1]
    assert np.float32(ce) > 0 and np.float32(cm) > 0
