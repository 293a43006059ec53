"""The reference's own acceptance runner with every JIT'd operator on the B200.

oracle/_ref/acceptance is proj/tests/acceptance.cpp compiled unmodified
against the reference library (oracle/Makefile). Its ten criteria
(acceptance.cpp:486-535) build operators through Operator::lower/apply, and
every one of those compiles through the toolchain seam of jit.cpp:84-95:
with STENCILFORGE_CC=bin/sf-cuda-cc the acoustic and diffusion operators bind
to libsf_b200.so's kernels and anything else is translated to CUDA
(paper_1609_03361_b200/cuda_cc.py). The runner then checks the GPU results
against its own naive interpreter, golden sources, dot tests and thread-count
bit-identity, exactly as it does for gcc.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNNER = os.path.join(ROOT, "oracle", "_ref", "acceptance")

pytestmark = pytest.mark.gpu


def test_reference_acceptance_through_sf_cuda_cc(tmp_path):
    if not os.path.exists(RUNNER):
        pytest.fail("oracle/_ref/acceptance not built (python -c 'import __graft_entry__ as g; "
                    "g.build()' in the container with /root/reference)")
    log = tmp_path / "cc.log"
    env = dict(os.environ, STENCILFORGE_CC=os.path.join(ROOT, "bin", "sf-cuda-cc"),
               SF_CUDA_CC_LOG=str(log))
    r = subprocess.run([RUNNER], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "acceptance_gpu.log"), "w") as f:
        f.write(out)
        if log.exists():
            f.write("\n# operators built by sf-cuda-cc\n" + log.read_text())
    passed = re.findall(r"\[PASS\] criterion\s+(\d+)", out)
    assert r.returncode == 0, out
    assert sorted(int(p) for p in passed) == list(range(1, 11)), out
    kinds = [line.split()[0] for line in log.read_text().splitlines()]
    # the GPU toolchain really built the operators: the recognised hot path
    # (acoustic, diffusion) went to the tuned kernels
    assert "acoustic" in kinds and "diffusion" in kinds, kinds
