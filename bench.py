"""Benchmark of the B200 stencil hot path (contract: one JSON line on rank 0).

Workload (default): BASELINE.json configs[1] (SURVEY "C2"), the 3D acoustic
forward at space order 4 on 281^3 (201^3 + 40-point damping layer on every
face), 10 m spacing, two layers 1.5/2.5 km/s, 10 Hz Ricker source at depth
20 m, 101 receivers on a line, 1000 ms at dt = 0.4 h / vmax = 1.6 ms
(625 steps). A benchmark "step" is one full apply of that operator: 625 time
steps of stencil + injection + sampling, i.e. 277^3 * 625 = 1.328e10
interior grid-point updates.

  value : GPts/s with every buffer resident in HBM (sf_plan_run, CUDA graph),
          device-timed with CUDA events, max over ranks.
  e2e   : GPts/s through the C-ABI entry sf_acoustic_apply with host (pinned)
          buffers: H2D of all nine arguments, the 625 steps, D2H of the three
          field slots and both traces, every step.
  roofline : the stencil kernel's algorithmic bytes (20 B per interior point:
          read u(t), u(t-1), m, eta, write u(t+1)) / its average launch time.

`--impl reference` times the reference's own CPU implementation (the
stencilforge library compiled from its sources into oracle/_ref, generated
C/OpenMP kernel via Operator::apply) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # SURVEY C1 / BASELINE configs[0]: 2D diffusion, exact 1/4 weights
    "c1": dict(kind="diffusion", n=2048, nt=500, order=2),
    # SURVEY C4 at one GPU: the 1024^3 per-GPU slab, order 8, 8 sources
    "c4": dict(shape=(1024, 1024, 1024), order=8, nt=1000, boundary=40, spacing=10.0,
               random=True, smooth="sines", nsrc=8),
    # FWI gradient, forward with full history + adjoint/gradient
    "c5": dict(kind="fwi", shape=(301, 301, 301), order=8, nt=1000, boundary=40, spacing=10.0),
    # SURVEY C2 / BASELINE configs[1]
    "c2": dict(shape=(281, 281, 281), order=4, nt=625, boundary=40, spacing=10.0,
               v_top=1500.0, v_bottom=2500.0, random=False),
    # SURVEY C3 / BASELINE configs[2] (one order per run)
    "c3o4": dict(shape=(512, 512, 512), order=4, nt=500, boundary=40, spacing=10.0,
                 random=True),
    "c3o6": dict(shape=(512, 512, 512), order=6, nt=500, boundary=40, spacing=10.0,
                 random=True),
    "c3o8": dict(shape=(512, 512, 512), order=8, nt=500, boundary=40, spacing=10.0,
                 random=True),
    "c3o12": dict(shape=(512, 512, 512), order=12, nt=500, boundary=40, spacing=10.0,
                  random=True),
    "c3o16": dict(shape=(512, 512, 512), order=16, nt=500, boundary=40, spacing=10.0,
                  random=True),
}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def smooth_velocity(shape, seed, sigma=8.0, vmin=1500.0, vmax=4500.0):
    """Seeded N(0,1) noise, separable Gaussian filter (sigma cells, truncate
    4 sigma, reflect), affinely rescaled to [vmin, vmax]."""
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal(shape, dtype=np.float32)
    f = gaussian_filter(noise, sigma=sigma, mode="reflect", truncate=4.0)
    lo, hi = float(f.min()), float(f.max())
    return vmin + (vmax - vmin) * (f.astype(np.float64) - lo) / (hi - lo)


def smooth_velocity_sines(shape, seed, vmin=1500.0, vmax=4500.0, modes=6):
    """Cheap smooth random velocity for very large grids (C4): a seeded sum
    of separable sinusoids with wavelengths >= 40 cells, rescaled to
    [vmin, vmax]. Built per plane (float64 only for one plane at a time)."""
    rng = np.random.default_rng(seed)
    n0, n1, n2 = shape
    k = rng.uniform(2 * np.pi / 200, 2 * np.pi / 40, (modes, 3))
    ph = rng.uniform(0, 2 * np.pi, (modes, 3))
    amp = rng.uniform(0.5, 1.0, modes)
    f1 = [np.cos(k[i, 1] * np.arange(n1) + ph[i, 1]) for i in range(modes)]
    f2 = [np.cos(k[i, 2] * np.arange(n2) + ph[i, 2]) for i in range(modes)]
    f0 = [np.cos(k[i, 0] * np.arange(n0) + ph[i, 0]) for i in range(modes)]
    tot = float(amp.sum())
    v = np.empty(shape, np.float64)
    for a in range(n0):
        pl = np.zeros((n1, n2))
        for i in range(modes):
            pl += amp[i] * f0[i][a] * np.outer(f1[i], f2[i])
        v[a] = vmin + (vmax - vmin) * (pl / tot + 1.0) * 0.5
    return v


def make_model(cfg_name):
    import paper_1609_03361_b200 as sf
    c = CONFIGS[cfg_name]
    shape = c["shape"]
    bw, h = c["boundary"], c["spacing"]
    if not c["random"]:
        vmax = max(c["v_top"], c["v_bottom"])
        model = sf.AcousticModel(shape=shape, boundary_width=bw, spacing=h, nt=c["nt"],
                                 space_order=c["order"], f0=10.0, v_top=c["v_top"],
                                 v_bottom=c["v_bottom"])
        model.dt = 0.4 * h / vmax
        mid = shape[1] // 2
        model.src_coords = [[(bw + 2) * h, mid * h, mid * h]]
        model.rec_coords = [[(bw + 2) * h, mid * h, (bw + 2 * i) * h] for i in range(101)]
        return model, None, None
    model = sf.AcousticModel(shape=shape, boundary_width=bw, spacing=h, nt=c["nt"],
                             space_order=c["order"], f0=10.0, v_top=4500.0, v_bottom=4500.0)
    model.dt = min(0.4 * h / 4500.0, model.stable_dt())
    mid = shape[1] // 2
    if c.get("nsrc", 1) > 1:  # C4: seeded random interior source positions
        rng = np.random.default_rng(8)
        r = c["order"] // 2
        model.src_coords = [[rng.uniform(bw + r, e - bw - r - 1) * h for e in shape]
                            for _ in range(c["nsrc"])]
        model.rec_coords = [[(bw + 10) * h, (bw + 2 + 7.3 * i) * h, mid * h] for i in range(101)]
        return model, smooth_velocity_sines(shape, 1234), 1500.0
    model.src_coords = [[(bw + 2) * h, mid * h, mid * h]]
    lo, hi = (bw + 2) * h, (shape[1] - bw - 3) * h
    g = np.linspace(lo + 0.37 * h, hi - 0.41 * h, 256)
    model.rec_coords = [[(bw + 10) * h, y, z] for y in g for z in g]
    return model, smooth_velocity(shape, 1234), 1500.0


def interior_points(model):
    r = model.space_order // 2
    n = 1
    for e in model.shape:
        n *= e - 2 * r
    return n


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                smax = float(p[1])
            except ValueError:
                continue
            for nm, val in zip(names, p[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_sample(model, cfg_name, v_field, v_min, steps=1, warmup=1, budget_s=20.0):
    """The reference's CPU path (oracle/_ref: stencilforge JIT kernel) on a
    bounded sample: the full grid for nt_s time steps. Returns GPts/s."""
    # SURVEY 8(d) CPU protocol: all host threads, pinned close to cores
    # (read by libgomp when the reference library loads it)
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    if ol.have_ref():
        ref = ol.Ref()
        kind = "reference"
        threads = ref.max_threads()
        ref.set_threads(threads)
        case = ol.AcousticCase(shape=model.shape, nt=1, boundary_width=model.boundary_width,
                               spacing=model.spacing, dt=model.dt, space_order=model.space_order,
                               f0=model.f0, v_top=model.v_top, v_bottom=model.v_bottom,
                               src_coords=model.src_coords, rec_coords=model.rec_coords)
        # calibrate: time a short run, then size the sample to the budget
        def timed(nt_s):
            case.nt = nt_s
            op = ol.ref_acoustic(ref, case, True)
            if v_field is not None:
                port = ol.Port()
                m, eta = port.medium_from_velocity(v_field, model.boundary_width, model.spacing,
                                                   v_min)
                op.set("m", m)
                op.set("eta", eta)
            op.build()
            t0 = time.perf_counter()
            op.apply()
            return time.perf_counter() - t0
        t_cal = timed(4)
        nt_s = int(max(4, min(model.nt, budget_s / max(t_cal / 4, 1e-6))))
        for _ in range(warmup):
            timed(min(nt_s, 4))
        times = [timed(nt_s) for _ in range(max(1, steps))]
        secs = float(np.median(times))
    else:
        port = ol.Port()
        kind = "port"
        import multiprocessing
        threads = multiprocessing.cpu_count()
        nt_s = 8
        m = np.zeros(model.shape, np.float32)
        eta = np.zeros_like(m)
        c = port.coefs(3, model.space_order, True, model.dt, model.spacing)
        u = np.zeros((3,) + tuple(model.shape), np.float32)
        src_ci, src_w = port.interp(np.array(model.src_coords), model.spacing, model.shape)
        rec_ci, rec_w = port.interp(np.array(model.rec_coords), model.spacing, model.shape)
        src = np.ones((nt_s, len(src_ci)), np.float32)
        rec = np.zeros((nt_s, len(rec_ci)), np.float32)
        t0 = time.perf_counter()
        port.acoustic_run(c, u, m + 1.0, eta, src, src_ci, src_w, rec, rec_ci, rec_w, nt_s)
        secs = time.perf_counter() - t0
    gpts = interior_points(model) * nt_s / secs / 1e9
    sample = (f"{cfg_name} grid {'x'.join(map(str, model.shape))} order {model.space_order}, "
              f"{nt_s} of {model.nt} time steps, median of {max(1, steps)} applies after "
              f"{warmup} warm-up, JIT excluded, OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')} "
              f"OMP_PLACES={os.environ.get('OMP_PLACES')}")
    return {"value": gpts, "unit": "GPts/s", "cores": threads, "kind": kind, "sample": sample}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    if CONFIGS[args.config].get("kind") == "diffusion":
        c = CONFIGS[args.config]
        base = cpu_diffusion_sample(c["n"], c["nt"], args.cpu_budget)
        pts = (c["n"] - 2) ** 2
        print(json.dumps({"impl": "reference", "metric": "GPts/s (grid-point updates/sec)",
                          "value": base["value"], "unit": "GPts/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": pts * c["nt"] / (base["value"] * 1e9) * 1e3,
                          "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic", "config": diffusion_config_block(c),
                          "cpu_baseline": base,
                          "e2e": {"value": base["value"], "unit": "GPts/s",
                                  "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    if CONFIGS[args.config].get("kind") == "fwi":
        print(json.dumps({"impl": "reference", "unavailable":
                          "the reference has no FWI gradient (SPEC.md:635,639)"}), flush=True)
        return
    model, v, vmin = make_model(args.config)
    base = cpu_reference_sample(model, args.config, v, vmin, steps=args.steps,
                                warmup=args.warmup, budget_s=args.cpu_budget)
    line = {
        "impl": "reference", "metric": "GPts/s (grid-point updates/sec)", "value": base["value"],
        "unit": "GPts/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        # one bench step = one full apply (all nt time steps) at the sampled rate
        "ms_per_step": interior_points(model) * model.nt / (base["value"] * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": config_block(args, model),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "GPts/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def diffusion_config_block(c):
    n, nt = c["n"], c["nt"]
    return {"workload": f"c1: 2D diffusion {n}^2, order 2, {nt} steps, alpha 1/2, "
                        f"dx 1/{n - 1}, dt = dx^2/4", "interior_points": (n - 2) ** 2,
            "l2": "2 x 16 MiB slots are L2-resident (126 MB L2); HBM roofline is "
                  "a lower bound here"}


def config_block(args, model):
    c = CONFIGS[args.config]
    return {"workload": f"{args.config}: 3D acoustic forward, space order {model.space_order}, "
                        f"{'x'.join(map(str, model.shape))} (boundary {c['boundary']}), "
                        f"{model.nt} time steps, dt {model.dt:.6g} s, "
                        f"{len(model.rec_coords)} receivers",
            "grid": list(model.shape), "space_order": model.space_order, "nt": model.nt,
            "interior_points": interior_points(model), "parallelism": f"replicas{args.gpus}",
            "l2": "working set (3 u slots + m + eta) larger than the 126 MB L2; no flush needed"}


def run_b200_arm(args, world, rank, local):
    import paper_1609_03361_b200 as sf
    model, v, vmin = make_model(args.config)
    setup = sf.acoustic_build(model, True, device=local, v_field=v, v_min=vmin, pinned=True)
    op = setup.op
    pts = interior_points(model)
    r = model.space_order // 2
    # resident: upload once, warm up (graph capture + clocks), then time
    op.upload()
    for _ in range(args.warmup):
        op.run(0, model.nt)
    op.synchronize()
    tot_ms, sten_ms, launches_per_run = op.time(stencil=True)
    import torch
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    barrier(world)
    with ClockSampler(local) as clocks:
        evs = []
        torch.cuda.synchronize()
        barrier(world)
        t_wall = time.perf_counter()
        total = 0.0
        for _ in range(args.steps):
            t, _, _ = op.time(stencil=False)
            total += t
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier(world)
    ms_per_step = max_over_ranks(world, total / args.steps)
    value = world * pts * model.nt / (ms_per_step / 1e3) / 1e9
    # average launch duration of the dominant kernel over the timed region:
    # the timed per-step time x the stencil's share of a run, the share from
    # a full run and a stencil-only run timed back to back right after the
    # timed region (same power / clock state; the share is ~0.99 because the
    # sparse work rides in the stencil's epilogue)
    tot2, sten2, _ = op.time(stencil=True)
    share = min(1.0, sten2 / tot2) if tot2 > 0 else 1.0
    stencil_launch_ms = ms_per_step / model.nt * share
    # compulsory bytes: read u(t), u(t-1), m, eta, write u(t+1) = 20 B/pt,
    # less the eta boxes the kernel skips because they are all zero (the
    # undamped interior) -- those bytes are not needed, so they are not
    # counted as achieved bandwidth
    eta_skip = op.eta_skip_fraction()
    alg_bytes = (20 - 4 * eta_skip) * pts
    peak, peak_kind = load_peaks()
    achieved = alg_bytes / (stencil_launch_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None
    # e2e through the C-ABI apply with pinned host buffers
    h2d = sum(a.data.nbytes for a in op.args)
    # apply returns what the kernel writes: the three slots and the receiver traces
    d2h = setup.field.data.nbytes + setup.rec.data.data.nbytes
    op.apply()  # warm
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.apply()
    e2e_s = max_over_ranks(world, (time.perf_counter() - t0) / args.steps)
    e2e = world * pts * model.nt / e2e_s / 1e9
    if rank != 0:
        return
    base = None
    if not args.no_cpu_baseline and world == 1:
        try:
            base = cpu_reference_sample(model, args.config, v, vmin, steps=1, warmup=1,
                                        budget_s=args.cpu_budget)
        except Exception as e:  # reported, not fatal
            base = {"error": str(e)}
    line = {
        "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(args, model),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_kind,
                     "kernel": f"3D stencil (radius {r}) avg launch {stencil_launch_ms * 1e3:.1f} us",
                     "alg_bytes_per_launch": alg_bytes, "eta_boxes_skipped": eta_skip},
        # second lens for the high orders: the reference's exact fp32 operation
        # count (no FMA contraction: 17 + 13r mul/add with c_j*temp3 shared
        # across the 6 neighbours of one offset, + 4 for the correctly rounded
        # reciprocal) against the non-FMA fp32 rate, 148 SMs x 128 lanes x clock
        "compute_roofline": {
            "bound": "fp32", "ops_per_point": 21 + 13 * r,
            "achieved": (21 + 13 * r) * pts / (stencil_launch_ms / 1e3) / 1e12,
            "peak": 148 * 128 * 1.965e9 / 1e12, "unit": "Tops/s",
            "frac": (21 + 13 * r) * pts / (stencil_launch_ms / 1e3) / (148 * 128 * 1.965e9),
            "peak_source": "148 SMs x 128 fp32 lanes x 1965 MHz (max SM clock)"},
        "stencil_share": share,
        "cpu_baseline": base,
        "e2e": {"value": e2e, "unit": "GPts/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches_per_run * args.steps),
        "clocks": clocks.summary(),
        "wall_s_timed_region": t_wall,
    }
    print(json.dumps(line), flush=True)


def run_b200_diffusion(args, world, rank, local):
    """C1: 2048^2 diffusion, alpha 1/2, dx 1/2047, dt = dx^2/4 (weights exactly
    1/4), 500 steps, seeded U[0,1) interior. 2 x 16 MiB slots: L2-resident."""
    from fractions import Fraction

    import paper_1609_03361_b200 as sf
    c = CONFIGS[args.config]
    n, nt = c["n"], c["nt"]
    cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(1, 2), dx=Fraction(1, n - 1),
                             dy=Fraction(1, n - 1), nt=nt, order=c["order"])
    b = sf.make_diffusion_operator(cfg, device=local, pinned=True)
    rng = np.random.default_rng(2016)
    u0 = np.zeros((n, n), np.float32)
    u0[1:-1, 1:-1] = rng.random((n - 2, n - 2))
    b.u.data[0] = u0
    b.u.data[1] = u0
    op = b.op
    op.upload()
    for _ in range(args.warmup):
        op.run(0, nt)
    op.synchronize()
    pts = (n - 2) ** 2
    with ClockSampler(local) as clocks:
        total = 0.0
        for _ in range(args.steps):
            t, _, nl = op.time(stencil=False)
            total += t
    ms = total / args.steps
    value = pts * nt / (ms / 1e3) / 1e9
    launch_ms = ms / nt
    peak, peak_kind = load_peaks()
    achieved = 8 * pts / (launch_ms / 1e3) / 1e9
    op.apply()
    # each apply uploads the pinned host slots, runs all nt steps and reads
    # both slots back in place; consecutive applies continue the run (the
    # work per apply is identical), so no host-side reset sits in the timed
    # region (re-filling 32 MiB of host memory per apply took ~3 ms)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.apply()
    e2e_s = (time.perf_counter() - t0) / args.steps
    base = None
    if not args.no_cpu_baseline:
        base = cpu_diffusion_sample(n, nt, args.cpu_budget)
    line = {
        "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": diffusion_config_block(c),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
                     "kernel": f"diffusion_tb_kernel (temporal blocking, T=8 steps per "
                               f"launch), {launch_ms * 1e3:.2f} us per time step",
                     "alg_bytes_per_launch": 8 * pts,
                     "note": "achieved = 8 B/pt per time step over the time per step; the "
                             "field is L2-resident, so HBM does not bind"},
        "cpu_baseline": base,
        "e2e": {"value": pts * nt / e2e_s / 1e9, "unit": "GPts/s",
                "h2d_bytes_per_step": b.u.data.nbytes, "d2h_bytes_per_step": b.u.data.nbytes},
        "gpu_launches": int(nl * args.steps), "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def cpu_diffusion_sample(n, nt, budget_s):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    rng = np.random.default_rng(2016)
    u0 = np.zeros((n, n), np.float32)
    u0[1:-1, 1:-1] = rng.random((n - 2, n - 2))
    if ol.have_ref():
        ref = ol.Ref()
        ref.set_threads(ref.max_threads())
        def timed(k):
            op = ol.ref_diffusion(ref, n, n, (1, 2), (1, n - 1), k, 2)
            op.set("u", np.stack([u0, u0]))
            op.build()
            t = time.perf_counter()
            op.apply()
            return time.perf_counter() - t
        cal = timed(10)
        k = int(max(10, min(nt, budget_s / max(cal / 10, 1e-6))))
        secs = timed(k)
        kind, cores = "reference", ref.max_threads()
    else:
        port = ol.Port()
        import multiprocessing
        k = 20
        u = np.stack([u0, u0])
        t = time.perf_counter()
        port.diffusion_run(u, 2, (1, 2), (1, n - 1), k)
        secs = time.perf_counter() - t
        kind, cores = "port", multiprocessing.cpu_count()
    return {"value": (n - 2) ** 2 * k / secs / 1e9, "unit": "GPts/s", "cores": cores,
            "kind": kind, "sample": f"c1 {n}^2 diffusion, {k} of {nt} steps, JIT excluded"}


def run_b200_fwi(args, world, rank, local):
    """C5: forward with the full wavefield history in HBM (nt+2 levels of
    301^3), adjoint injecting seeded N(0,1) residuals at 201 x 201 surface
    receivers, gradient accumulated in the adjoint stencil. The metric counts
    the updates of both passes."""
    import paper_1609_03361_b200 as sf
    c = CONFIGS[args.config]
    shape, order, nt, bw, h = c["shape"], c["order"], c["nt"], c["boundary"], c["spacing"]
    r = order // 2
    v = smooth_velocity(shape, 1234)
    g = sf.Grid()
    model = sf.AcousticModel(shape=shape, boundary_width=bw, spacing=h, nt=nt,
                             space_order=order, v_top=4500.0, v_bottom=4500.0)
    dt = min(0.4 * h / 4500.0, model.stable_dt())
    m, eta = sf.build_medium(g, model, v_field=v, v_min=1500.0)
    mid = shape[1] // 2
    src_c = [[(bw + 2) * h, mid * h, mid * h]]
    rec_c = [[(bw + 10) * h, (bw + i) * h, (bw + j) * h] for i in range(201) for j in range(201)]
    def interp(coords):
        cis, ws = zip(*[sf.interpolation_weights(cc, h, shape) for cc in coords])
        return np.array(cis, np.int32), np.array(ws, np.float32)
    src_ci, src_w = interp(src_c)
    rec_ci, rec_w = interp(rec_c)
    t0 = 1.0 / 10.0
    src = np.array([sf.ricker_wavelet(10.0, t * dt, t0) for t in range(nt)], np.float32)[:, None]
    rng = np.random.default_rng(5)
    residual = rng.standard_normal((nt, len(rec_c)), dtype=np.float32)
    plan = sf.FwiPlan(shape, order, nt, dt, h, 1, len(rec_c), device=local)
    # warm-up call (graph capture, sparse index build), then the timed one
    plan.gradient(m.data, eta.data, src, src_ci, src_w, rec_ci, rec_w, residual)
    t_e = time.perf_counter()
    rec_out, grad, _, _ = plan.gradient(m.data, eta.data, src, src_ci, src_w, rec_ci, rec_w,
                                        residual)
    e2e_s = time.perf_counter() - t_e
    fwd = adj = 0.0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            f, a = plan.time()
            fwd += f
            adj += a
    fwd /= args.steps
    adj /= args.steps
    pts = 1
    for e in shape:
        pts *= e - 2 * r
    value = 2 * pts * nt / ((fwd + adj) / 1e3) / 1e9
    peak, peak_kind = load_peaks()
    # the all-zero eta boxes both sweeps skip (the forward tiling's fraction,
    # applied to both) are not counted as achieved bytes
    skip = plan.eta_skip_fraction()
    bf, ba = 20 - 4 * skip, 36 - 4 * skip
    line = {
        "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
        "n_gpus": 1, "steps": args.steps, "warmup": 1, "ms_per_step": fwd + adj,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"c5: FWI gradient {shape[0]}^3, order {order}, {nt} steps, "
                               f"history {nt + 2} levels in HBM, {len(rec_c)} receivers",
                   "forward_ms": fwd, "adjoint_gradient_ms": adj,
                   "grad_abs_max": float(np.abs(grad).max())},
        "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_kind,
                     "forward_achieved": bf * pts * nt / (fwd / 1e3) / 1e9,
                     "adjoint_achieved": ba * pts * nt / (adj / 1e3) / 1e9,
                     "achieved": (bf + ba) * pts * nt / ((fwd + adj) / 1e3) / 1e9,
                     "frac": (bf + ba) * pts * nt / ((fwd + adj) / 1e3) / 1e9 / peak,
                     "traffic": None, "eta_boxes_skipped": skip},
        "e2e": {"value": 2 * pts * nt / e2e_s / 1e9, "unit": "GPts/s",
                "h2d_bytes_per_step": m.data.nbytes * 2 + residual.nbytes + src.nbytes,
                "d2h_bytes_per_step": grad.nbytes + rec_out.nbytes},
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_b200_slabs(args, world, rank, local):
    """N > 1: weak scaling over depth slabs. The global grid stacks one c2-sized
    block per GPU along axis 0 ((281 N) x 281 x 281, same boundary, source and
    receiver line at the top); rank g owns 281 planes and swaps r-deep halos
    with its neighbours over NCCL inside every time step (sf_plan_attach_nccl)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200 import _lib
    from paper_1609_03361_b200.slab import SlabPartition, SlabRun, nccl_unique_id
    base, _, _ = make_model(args.config)
    if CONFIGS[args.config]["random"]:
        raise SystemExit("multi-GPU bench uses the c2 layered workload")
    r = base.space_order // 2
    gshape = (base.shape[0] * world,) + tuple(base.shape[1:])
    model = sf.AcousticModel(shape=gshape, boundary_width=base.boundary_width,
                             spacing=base.spacing, nt=base.nt, dt=base.dt,
                             space_order=base.space_order, f0=base.f0, v_top=base.v_top,
                             v_bottom=base.v_bottom, src_coords=base.src_coords,
                             rec_coords=base.rec_coords)
    g = sf.Grid()
    m, eta = sf.build_medium(g, model)
    src_ci = np.array([sf.interpolation_weights(c, model.spacing, gshape)[0]
                       for c in model.src_coords], np.int32)
    src_w = np.array([sf.interpolation_weights(c, model.spacing, gshape)[1]
                      for c in model.src_coords], np.float32)
    rec_ci = np.array([sf.interpolation_weights(c, model.spacing, gshape)[0]
                       for c in model.rec_coords], np.int32)
    rec_w = np.array([sf.interpolation_weights(c, model.spacing, gshape)[1]
                      for c in model.rec_coords], np.float32)
    t0 = 1.0 / model.f0
    ser = np.array([sf.ricker_wavelet(model.f0, t * model.dt, t0) for t in range(model.nt)],
                   np.float32)[:, None]
    rec = np.zeros((model.nt, len(rec_ci)), np.float32)
    part = SlabPartition.split(gshape[0], r, world, rank)
    slab = SlabRun(part, gshape, model.space_order, True, model.nt, model.dt, model.spacing,
                   m.data, eta.data, ser, src_ci, src_w, rec, rec_ci, rec_w, device=local)
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    slab.attach_nccl(obj[0], world, rank)
    for _ in range(args.warmup):
        slab.run(0, model.nt)
    barrier(world)
    tot = C.c_float()
    sten = C.c_float()
    nl = C.c_int64()
    with ClockSampler(local) as clocks:
        total = 0.0
        for _ in range(args.steps):
            sf.api.check(_lib.lib.sf_plan_time(slab.plan, C.byref(tot), None, C.byref(nl)))
            total += tot.value
    barrier(world)
    ms_per_step = max_over_ranks(world, total / args.steps)
    # per-rank stencil-only pass (no exchange) for the roofline of the kernel
    sf.api.check(_lib.lib.sf_plan_time(slab.plan, C.byref(tot), C.byref(sten), C.byref(nl)))
    sten_ms = max_over_ranks(world, sten.value)
    pts = 1
    for e in gshape:
        pts *= e - 2 * r
    value = pts * model.nt / (ms_per_step / 1e3) / 1e9
    # e2e: upload host slices, run, download, every step (pinned host buffers,
    # as in the single-GPU arm)
    def pinned(a):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        arr = t.numpy()
        arr[...] = a
        return arr, t
    keep = [pinned(b) for b in slab.bufs]
    slab.bufs = [k[0] for k in keep]
    barrier(world)
    t_e = time.perf_counter()
    for _ in range(args.steps):
        argv = (C.c_void_p * 9)(*[b.ctypes.data for b in slab.bufs])
        sf.api.check(_lib.lib.sf_plan_invoke(slab.plan, argv, 9))
    e2e_s = max_over_ranks(world, (time.perf_counter() - t_e) / args.steps)
    h2d = sum(b.nbytes for b in slab.bufs)
    d2h = slab.bufs[0].nbytes + slab.bufs[6].nbytes
    if rank == 0:
        line = {
            "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config} stacked along depth: "
                                   f"{'x'.join(map(str, gshape))}, order {model.space_order}, "
                                   f"{model.nt} steps, {world} depth slabs of "
                                   f"{base.shape[0]} planes, NCCL halo exchange ({r} planes) "
                                   "every step", "grid": list(gshape),
                       "parallelism": f"slab{world}", "interior_points": pts},
            "e2e": {"value": pts * model.nt / e2e_s / 1e9, "unit": "GPts/s",
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world},
            "gpu_launches": int(nl.value * args.steps),
            "clocks": clocks.summary(),
        }
        peak, peak_kind = load_peaks()
        own_pts = pts // world  # each rank updates its own slab's interior share
        import ctypes
        frac = ctypes.c_double()
        sf.api.check(_lib.lib.sf_plan_eta_skip_fraction(slab.plan, ctypes.byref(frac)))
        bpp = 20 - 4 * frac.value  # less the all-zero eta boxes the kernel skips
        achieved = bpp * own_pts / (sten_ms / model.nt / 1e3) / 1e9
        line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
                            "kernel": f"3D stencil (radius {r}) per rank, avg launch "
                                      f"{sten_ms / model.nt * 1e3:.1f} us (stencil-only pass)",
                            "alg_bytes_per_launch": bpp * own_pts,
                            "eta_boxes_skipped": frac.value}
        print(json.dumps(line), flush=True)
    slab.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # exercise the multi-GPU slab path (NCCL communicator, slab plans) with a
    # single rank: validates the N > 1 code on a one-GPU box
    ap.add_argument("--force-slabs", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_init(args)
    try:
        kind = CONFIGS[args.config].get("kind", "acoustic")
        if args.impl == "reference":
            run_reference_arm(args, world, rank)
        elif kind == "diffusion":
            if rank == 0:
                run_b200_diffusion(args, world, rank, local)
        elif kind == "fwi":
            if rank == 0:
                run_b200_fwi(args, world, rank, local)
        elif world > 1 or args.force_slabs:
            run_b200_slabs(args, world, rank, local)
        else:
            run_b200_arm(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
