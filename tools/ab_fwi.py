"""Interleaved A/B timing of FWI (C5) plan variants: forward sweep with the
history and the adjoint+gradient sweep, each variant a separate FwiPlan built
under its SF_* environment, timed round-robin in one process (same power
state). The history is (nt+2) levels of 301^3, so nt is reduced (default 250
steps, ~27 GB per plan); per-step times do not depend on nt.

    python tools/ab_fwi.py 5 250 "" "SF_ZCHUNKS=4" "SF_TMA_STAGES_GRAD=3"
"""
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    rounds, nt = int(sys.argv[1]), int(sys.argv[2])
    variants = sys.argv[3:]
    import paper_1609_03361_b200 as sf
    shape, order = (301, 301, 301), 8
    h, bw = bench.H, bench.BW
    dt = min(0.4 * h / 4500.0, sf.api._stable_dt(3, order, h, 4500.0, 4500.0))
    sm = sf.SmoothMedium(shape=shape, boundary_width=bw, spacing=h, **bench.SMOOTH)
    lo, hi = sm.extrema()
    m, eta = sm.generate(lo, hi)
    mid = shape[1] // 2
    src_c = [[(bw + 2) * h, mid * h, mid * h]]
    rec_c = [[(bw + 10) * h, (bw + i) * h, (bw + j) * h] for i in range(201) for j in range(201)]

    def interp(coords):
        cis, ws = zip(*[sf.interpolation_weights(cc, h, shape) for cc in coords])
        return np.array(cis, np.int32), np.array(ws, np.float32)
    sci, sw = interp(src_c)
    rci, rw = interp(rec_c)
    src = np.array([sf.ricker_wavelet(10.0, t * dt, 0.1) for t in range(nt)], np.float32)[:, None]
    res = np.random.default_rng(5).standard_normal((nt, len(rec_c)), dtype=np.float32)
    plans = []
    for var in variants:
        saved = dict(os.environ)
        for kv in filter(None, var.split(",")):
            k, val = kv.split("=", 1)
            os.environ[k] = val
        p = sf.FwiPlan(shape, order, nt, dt, h, 1, len(rec_c))
        p.gradient(m, eta, src, sci, sw, rci, rw, res)
        os.environ.clear()
        os.environ.update(saved)
        plans.append(p)
    tf = [[] for _ in variants]
    ta = [[] for _ in variants]
    for _ in range(rounds):
        for i, p in enumerate(plans):
            f, a = p.time()
            tf[i].append(f / nt * 1e3)
            ta[i].append(a / nt * 1e3)
    pts = bench.interior_points(shape, order)
    for var, f, a in zip(variants, tf, ta):
        mf, ma = statistics.median(f), statistics.median(a)
        print(json.dumps({"cfg": "c5", "variant": var, "fwd_us_per_step": mf, "adj_us_per_step": ma,
                          "fwd_gpts": pts / (mf * 1e-6) / 1e9, "adj_gpts": pts / (ma * 1e-6) / 1e9,
                          "c5_gpts": 2 * pts / ((mf + ma) * 1e-6) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
