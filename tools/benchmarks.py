"""The reference's benchmark helpers (bench.hpp / bench.cpp) on the B200.

`bench_acoustic` / `bench_diffusion` keep the reference's protocol
(bench.cpp:41-53): snapshot every host buffer, one untimed warm-up, then the
median of `runs` timed applies with the buffers restored before each run, one
`BenchLine` per variant, printed by `format_bench` in the reference's text
format. Where the reference sweeps CPU cache-blocking plans, the GPU sweeps its
kernel configurations (family x tile x pipeline depth, `Operator.autotune`):

* variant "apply"    — `Operator.apply` through host buffers (H2D + all steps
                       + D2H), the call a reference user times;
* variant "resident" — every kernel configuration on HBM-resident state
                       (plan = its description), as `Operator::autotune`
                       (op.cpp:169-221) times its candidates.
"""
from __future__ import annotations

import statistics
import time
from dataclasses import dataclass

import numpy as np

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_03361_b200 import api  # noqa: E402


@dataclass
class BenchLine:
    """bench.hpp:9-15"""
    scenario: str
    variant: str
    plan: str
    runs: int
    median_s: float


def _time_apply(scenario, runs, op, buffers):
    """run_variant (bench.cpp:41-53): warm-up, then median of restored runs."""
    snap = [b.copy() for b in buffers]

    def restore():
        for b, s in zip(buffers, snap):
            b[...] = s

    op.apply()  # warm-up (and graph capture), excluded
    times = []
    for _ in range(max(1, runs)):
        restore()
        t0 = time.perf_counter()
        op.apply()
        times.append(time.perf_counter() - t0)
    restore()
    return BenchLine(scenario, "apply", "default", runs, float(statistics.median(times)))


def bench_acoustic(model: api.AcousticModel, runs: int = 3, sweep: bool = True,
                   device: int = 0):
    """bench_acoustic (bench.cpp:96-119) for the forward operator."""
    cells = int(np.prod(model.shape))
    if exceeds_memory(cells * 4 * 7, device):  # 3 slots + m + eta + staging + slack
        return [BenchLine("acoustic", "apply", "SkippedTooLarge", 0, 0.0)]
    s = api.acoustic_forward(model, device=device)
    bufs = [a.data for a in s.op.args]
    out = [_time_apply("acoustic", runs, s.op, bufs)]
    if sweep:
        s.op.upload()
        rep, _ = s.op.autotune(tune_nt=model.nt, repeats=max(1, runs))
        out += [BenchLine("acoustic", "resident", desc, runs, t) for desc, t in rep]
    return out


def bench_diffusion(cfg: api.DiffusionConfig, runs: int = 3, device: int = 0):
    """bench_diffusion (bench.cpp:57-91): the reference's Gaussian-blob start
    (gaussian_blob_field) in slot 0, one line for the GPU apply."""
    b = api.make_diffusion_operator(cfg, device=device)
    b.u.data[0] = api.gaussian_blob_field(cfg.nx, cfg.ny)
    return [_time_apply("diffusion", runs, b.op, [b.u.data])]


def format_bench(lines) -> str:
    """format_bench (bench.cpp:121-133): one machine-readable line per variant."""
    return "".join(f"bench scenario={l.scenario} variant={l.variant} plan={l.plan} "
                   f"runs={l.runs} median_s={l.median_s:.6f}\n" for l in lines)


def exceeds_memory(nbytes: int, device: int = 0) -> bool:
    """exceeds_memory (bench.cpp:159-165), against the device's HBM: true when
    the footprint exceeds half of it."""
    import torch
    if not torch.cuda.is_available():
        return False
    total = torch.cuda.get_device_properties(device).total_memory
    return nbytes > total // 2
