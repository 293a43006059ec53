"""Sweep the 3D stencil tile shapes (SF_TILE=nx,ty) on one config and print
the average stencil launch time and achieved algorithmic GB/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    nt = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    tiles = sys.argv[3].split(";") if len(sys.argv) > 3 else [
        "1,8", "1,16", "2,8", "2,16", "3,8", "3,16", "4,8", "4,16"]
    import paper_1609_03361_b200 as sf
    w = bench.workload(cfg, 1, bench.product_stable_dt(sf))
    pts = bench.interior_points(w.shape, w.order)
    out = []
    for t in tiles:
        os.environ["SF_TILE"] = t
        try:
            s = bench.b200_setup(sf, w, nt=nt)
        except Exception as e:  # tile not compiled for this order
            print(cfg, t, "skip", e)
            continue
        s.op.upload()
        s.op.run(0, nt)
        s.op.synchronize()
        best = None
        for _ in range(3):
            tot, st, _ = s.op.time(stencil=True)
            best = st if best is None else min(best, st)
        us = best / nt * 1e3
        gbs = 20 * pts / (us * 1e-6) / 1e9
        rec = {"cfg": cfg, "tile": t, "stencil_us": us, "alg_GBps": gbs,
               "gpts": pts / (us * 1e-6) / 1e9}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del s


if __name__ == "__main__":
    main()
