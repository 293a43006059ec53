"""Interleaved A/B timing of stencil-kernel variants on one bench config.

The B200's power cap moves the SM clock between runs by up to ~20 %, which
swamps few-percent kernel changes measured in separate processes. Here every
variant (a set of SF_* environment knobs read at plan creation) gets its own
plan in ONE process, and the variants' full time loops are timed round-robin,
so they see the same thermal / power state; the median per variant is
reported. Usage:

    python tools/ab_time.py c2 20 "SF_VEC_RPL=1" "SF_VEC_RPL=2"
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    cfg = sys.argv[1]
    rounds = int(sys.argv[2])
    variants = sys.argv[3:]
    import paper_1609_03361_b200 as sf
    w = bench.workload(cfg, 1, bench.product_stable_dt(sf))
    nt = w.nt
    pts = bench.interior_points(w.shape, w.order)
    plans = []
    for var in variants:
        saved = dict(os.environ)
        for kv in filter(None, var.split(",")):
            k, val = kv.split("=", 1)
            os.environ[k] = val
        s = bench.b200_setup(sf, w)
        os.environ.clear()
        os.environ.update(saved)
        s.op.upload()
        s.op.run(0, nt)
        s.op.synchronize()
        plans.append(s)
    times = [[] for _ in variants]
    for _ in range(rounds):
        for i, s in enumerate(plans):
            tot, _, _ = s.op.time(stencil=False)
            times[i].append(tot / nt * 1e3)
    for var, t in zip(variants, times):
        med = statistics.median(t)
        print(json.dumps({"cfg": cfg, "variant": var, "us_per_step_median": med,
                          "us_min": min(t), "gpts": pts / (med * 1e-6) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
