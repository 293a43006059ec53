"""The reference-side C++ binding (integration/sf_cuda_backend.cpp): written
against stencilforge's public headers, it builds an sf_plan from a lowered
Operator's own metadata and applies it with the operator's buffers in
KernelSignature order -- what `CodegenConfig::preset == "cuda"` would do inside
the reference's op.cpp. integration/_build/backend_check runs the reference's
acoustic_build operators once through the JIT'd C (Operator::apply) and once
through the binding, and compares every grid buffer bitwise."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = os.path.join(ROOT, "integration", "_build", "backend_check")


def _run():
    if not os.path.exists(CHECK):
        pytest.fail("integration/_build/backend_check not built (__graft_entry__.build())")
    r = subprocess.run([CHECK], cwd=ROOT, capture_output=True, text=True, timeout=900)
    return r.returncode, [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]


def test_binding_fails_loudly_without_a_device():
    """No CPU fallback: without a B200 the binding raises the reference's
    CompileFailedError from sf_acoustic_plan_create (after the reference's own
    host apply ran)."""
    import paper_1609_03361_b200 as sf
    if sf._lib.lib.sf_device_count() > 0:
        pytest.skip("a CUDA device is present")
    if not os.path.exists(CHECK):
        pytest.skip("integration/_build not built (needs /root/reference; __graft_entry__.build())")
    rc, lines = _run()
    assert rc != 0
    assert lines and all("no CUDA device" in ln.get("error", "") for ln in lines)


@pytest.mark.gpu
def test_binding_bitwise_vs_reference_jit():
    rc, lines = _run()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "integration_binding.jsonl"), "w") as f:
        f.write("\n".join(json.dumps(x) for x in lines) + "\n")
    assert rc == 0, lines
    assert len(lines) == 6 and all(ln["mismatched"] == 0 and ln["buffers"] >= 9 for ln in lines)
