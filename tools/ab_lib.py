"""Interleaved A/B of two BUILDS of libsf_b200.so in one process.

Compile-time changes cannot be switched by an SF_* knob, and separate
processes see different power-cap states. This loads the package twice — the
in-tree build, and a renamed copy of the package whose libsf_b200.so is the
given alternate build — creates one plan per (build, knob set) and times their
full time loops round-robin. Usage:

    python tools/ab_lib.py /path/to/base.so c3o16 12 ["SF_X=1" ...]

Variants are reported as base:<knobs> and new:<knobs>.
"""
import importlib
import json
import os
import shutil
import statistics
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def load_alt(so_path):
    d = tempfile.mkdtemp(prefix="sf_ab_")
    pkg = os.path.join(d, "sf_b200_base")
    os.makedirs(pkg)
    src = os.path.join(ROOT, "paper_1609_03361_b200")
    for f in os.listdir(src):
        if f.endswith(".py"):
            shutil.copy(os.path.join(src, f), pkg)
    shutil.copy(so_path, os.path.join(pkg, "libsf_b200.so"))
    sys.path.insert(0, d)
    return importlib.import_module("sf_b200_base")


def main():
    base_so, cfg, rounds = sys.argv[1], sys.argv[2], int(sys.argv[3])
    knobs = sys.argv[4:] or [""]
    import paper_1609_03361_b200 as sf_new
    sf_base = load_alt(base_so)
    w = bench.workload(cfg, 1, bench.product_stable_dt(sf_new))
    nt = w.nt
    pts = bench.interior_points(w.shape, w.order)
    plans, names = [], []
    for var in knobs:
        for tag, sf in (("base", sf_base), ("new", sf_new)):
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
            names.append(f"{tag}:{var}")
    times = [[] for _ in plans]
    for _ in range(rounds):
        for i, s in enumerate(plans):
            tot, _, _ = s.op.time(stencil=False)
            times[i].append(tot / nt * 1e3)
    for name, t in zip(names, times):
        med = statistics.median(t)
        print(json.dumps({"cfg": cfg, "variant": name, "us_per_step_median": round(med, 2),
                          "us_min": round(min(t), 2),
                          "gpts": round(pts / (med * 1e-6) / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
