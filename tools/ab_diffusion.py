"""Interleaved A/B timing of diffusion (C1) plan variants (SF_* knobs read at
plan creation), like paper_1609_03361_b200/ab_time.py for the acoustic configs.
    python tools/ab_diffusion.py 10 "" "SF_TB_TILE=72" "SF_TB_TILE=96"
"""
import json
import os
import statistics
import sys
from fractions import Fraction

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_03361_b200 as sf  # noqa: E402


def main():
    rounds = int(sys.argv[1])
    variants = sys.argv[2:]
    n, nt = 2048, 500
    ops = []
    for var in variants:
        saved = dict(os.environ)
        for kv in filter(None, var.split(",")):
            k, val = kv.split("=", 1)
            os.environ[k] = val
        cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(1, 2), dx=Fraction(1, n - 1),
                                 dy=Fraction(1, n - 1), nt=nt, order=2)
        b = sf.make_diffusion_operator(cfg, device=0, pinned=True)
        os.environ.clear()
        os.environ.update(saved)
        rng = np.random.default_rng(2016)
        u0 = np.zeros((n, n), np.float32)
        u0[1:-1, 1:-1] = rng.random((n - 2, n - 2))
        b.u.data[0] = u0
        b.u.data[1] = u0
        b.op.apply()  # the result for the parity check below
        ops.append(b)
    ref = ops[0].u.data.copy()
    for var, b in zip(variants, ops):
        assert np.array_equal(b.u.data.view(np.uint32), ref.view(np.uint32)), var
        b.op.upload()
        b.op.run(0, nt)
        b.op.synchronize()
    times = [[] for _ in variants]
    for _ in range(rounds):
        for i, b in enumerate(ops):
            t, _, _ = b.op.time(stencil=False)
            times[i].append(t / nt * 1e3)
    pts = (n - 2) ** 2
    for var, t in zip(variants, times):
        med = statistics.median(t)
        print(json.dumps({"cfg": "c1", "variant": var, "us_per_step_median": med,
                          "gpts": pts / (med * 1e-6) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
