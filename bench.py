"""Benchmark of the B200 stencil hot path (contract: one JSON line on rank 0).

Default workload: SURVEY C4 at one GPU -- the largest single-GPU config of
BASELINE.json: 3D acoustic forward, space order 8, 1024^3 (40-point damping
layer on every face), 10 m spacing, seeded smooth random velocity in
[1.5, 4.5] km/s (Gaussian-filtered noise, sigma 8 cells, generated on the GPU
from global indices: csrc/medium.cu), 8 Ricker sources at seeded random
positions, 101 receivers, 1000 time steps at dt = 0.4 h / vmax. With
`--gpus N` (torchrun) the grid is N such blocks stacked in depth
((1024 N) x 1024 x 1024), one depth slab per GPU, r-deep halos exchanged over
NCCL every step, each rank generating only its own slab's medium (weak
scaling). `--config` selects the other BASELINE configs (c1 diffusion, c2,
c3o4..c3o16, c5 FWI). A bench "step" is one full apply: all nt time steps of
stencil + injection + sampling.

  value : GPts/s with every buffer resident in HBM (sf_plan_run, CUDA graph),
          device-timed with CUDA events, max over ranks.
  e2e   : GPts/s through the C-ABI entry sf_plan_invoke (Operator.apply)
          with pinned host buffers: H2D of all nine arguments, the nt steps,
          D2H of the three field slots and the traces, every step.
  roofline : the stencil kernel's algorithmic bytes (20 B per interior point:
          read u(t), u(t-1), m, eta, write u(t+1), less the all-zero eta
          boxes the kernel skips) / its average launch time.

`--impl reference` times the reference's own CPU implementation (stencilforge
compiled from its sources into oracle/_ref: acoustic_build + the JIT'd
C/OpenMP Operator::apply) on a bounded sample of the same workload. That arm
never imports this package (it uses only oracle/ through tests/oracle_lib).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SMOOTH = dict(seed=1234, sigma=8.0, v_lo=1500.0, v_hi=4500.0, v_min=1500.0)

CONFIGS = {
    # SURVEY C4 at one GPU (default): the 1024^3 per-GPU block, order 8, 8 sources
    "c4": dict(shape=(1024, 1024, 1024), order=8, nt=1000, nsrc=8, recs="line"),
    # SURVEY C1 / BASELINE configs[0]: 2D diffusion, exact 1/4 weights
    "c1": dict(kind="diffusion", n=2048, nt=500, order=2),
    # FWI gradient, forward with full history + adjoint/gradient
    "c5": dict(kind="fwi", shape=(301, 301, 301), order=8, nt=1000),
    # SURVEY C2 / BASELINE configs[1]: two layers 1.5 / 2.5 km/s
    "c2": dict(shape=(281, 281, 281), order=4, nt=625, layered=True),
    # SURVEY C3 / BASELINE configs[2] (one order per run), 256 x 256 receivers
    **{f"c3o{o}": dict(shape=(512, 512, 512), order=o, nt=500, recs="surface")
       for o in (4, 6, 8, 10, 12, 14, 16)},
}
BW, H = 40, 10.0


def workload(name, world=1, stable_dt=None):
    """The acoustic workload of a config, global over `world` depth blocks.
    stable_dt(order, v_max) -> seconds is supplied by the caller (the product's
    or the reference's own AcousticModel::stable_dt), so this function needs
    neither implementation."""
    c = CONFIGS[name]
    block = tuple(c["shape"])
    shape = (block[0] * world,) + block[1:]
    order, nt = c["order"], c["nt"]
    r = order // 2
    mid = block[1] // 2
    w = SimpleNamespace(name=name, block=block, shape=shape, order=order, nt=nt, bw=BW, h=H,
                        f0=10.0, world=world)
    if c.get("layered"):
        w.v_top, w.v_bottom, w.smooth = 1500.0, 2500.0, None
        w.dt = 0.4 * H / 2500.0
        w.src_coords = [[(BW + 2) * H, mid * H, mid * H]]
        w.rec_coords = [[(BW + 2) * H, mid * H, (BW + 2 * i) * H] for i in range(101)]
        return w
    w.v_top = w.v_bottom = 4500.0
    w.smooth = dict(SMOOTH, shape=shape, boundary_width=BW, spacing=H)
    w.dt = min(0.4 * H / 4500.0, stable_dt(order, 4500.0))
    if c.get("nsrc", 1) > 1:  # C4: seeded random interior source positions (global grid)
        rng = np.random.default_rng(8)
        w.src_coords = [[rng.uniform(BW + r, e - BW - r - 1) * H for e in shape]
                        for _ in range(c["nsrc"])]
    else:
        w.src_coords = [[(BW + 2) * H, mid * H, mid * H]]
    if c.get("recs") == "line":
        w.rec_coords = [[(BW + 10) * H, (BW + 2 + 7.3 * i) * H, mid * H] for i in range(101)]
    else:
        lo, hi = (BW + 2) * H, (block[1] - BW - 3) * H
        g = np.linspace(lo + 0.37 * H, hi - 0.41 * H, 256)
        w.rec_coords = [[(BW + 10) * H, y, z] for y in g for z in g]
    return w


def interior_points(shape, order):
    r = order // 2
    n = 1
    for e in shape:
        n *= e - 2 * r
    return n


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_info():
    model, phys = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            cur = {}
            for ln in f:
                if ":" in ln:
                    k, v = [x.strip() for x in ln.split(":", 1)]
                    cur[k] = v
                    if k == "model name":
                        model = v
                elif cur:
                    phys.add((cur.get("physical id"), cur.get("core id")))
                    cur = {}
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(),
            "physical_cores": len(phys) if phys and None not in next(iter(phys)) else None}


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
            # a timed region shorter than nvidia-smi's start-up (C1: ~13 ms)
            # would leave no sample: take the first one it prints
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons, watts = [], None, set(), []
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
            try:
                watts.append(float(p[2]))
            except ValueError:
                pass
            for nm, val in zip(names, p[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
               "samples": len(sm)}
        if watts:
            out["power_w_median"] = float(np.median(watts))
        return out


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class stdout_to_stderr:
    """File descriptor 1 -> 2 for a block: library banners (NCCL prints its
    version at communicator init on some setups) must not land on stdout,
    which carries exactly one JSON line from rank 0."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_start(local):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_over_ranks(world, value, op="max"):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return float(t.item())


# ---------------------------------------------------------------------------
# The reference's CPU path (oracle/_ref, else the C port): never imports the
# B200 package.

def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    return ol


def _ref_threads():
    # SURVEY 8(d) CPU protocol: all host threads, pinned close to cores (read
    # by libgomp when the reference library loads it)
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")


def ref_acoustic_sample(w, budget_s, runs, warmup, forward_adjoint=False):
    """Median GPts/s of `runs` applies of the reference's acoustic operator
    (acoustic_build + Operator::apply, JIT'd OpenMP C, JIT excluded) on the
    workload's first depth block, nt_s time steps each (nt_s sized so that
    warmup + runs applies take about budget_s). forward_adjoint: each apply
    is the forward operator then the adjoint one (FWI's two sweeps, the
    gradient product itself excluded: the reference has none)."""
    _ref_threads()
    ol = _oracle()
    shape = w.block  # the reference has no decomposition: one block
    pts = interior_points(shape, w.order)
    if not ol.have_ref():
        raise RuntimeError("oracle/_ref/libsf_ref.so missing")
    ref = ol.Ref()
    threads = ref.max_threads()
    ref.set_threads(threads)
    medium = None
    t_med = None
    if w.smooth is not None:
        port = ol.Port()
        t0 = time.perf_counter()
        lo, hi = port.smooth_extrema(shape, 0, shape[0], w.smooth["seed"], w.smooth["sigma"])
        medium = port.smooth_medium(shape, 0, shape[0], w.smooth["seed"], lo, hi,
                                    sigma=w.smooth["sigma"], v_lo=w.smooth["v_lo"],
                                    v_hi=w.smooth["v_hi"], boundary_width=w.bw, spacing=w.h,
                                    v_min=w.smooth["v_min"])
        t_med = time.perf_counter() - t0
    # sources / receivers of the block (the slab workload keeps them in block 0)
    src = [c for c in w.src_coords if c[0] < (shape[0] - 1) * w.h] or w.src_coords[:1]

    def build(nt_s, forward=True):
        case = ol.AcousticCase(shape=shape, nt=nt_s, boundary_width=w.bw, spacing=w.h, dt=w.dt,
                               space_order=w.order, f0=w.f0, v_top=w.v_top,
                               v_bottom=w.v_bottom, src_coords=src, rec_coords=w.rec_coords)
        op = ol.ref_acoustic(ref, case, forward)
        if medium is not None:
            op.set("m", medium[0])
            op.set("eta", medium[1])
        op.build()
        return op

    def apply_all(ops):
        t0 = time.perf_counter()
        for o in ops:
            o.apply()
        return time.perf_counter() - t0

    ops = [build(1, True)] + ([build(1, False)] if forward_adjoint else [])
    apply_all(ops)
    t1 = apply_all(ops)
    nt_s = int(max(1, min(w.nt, round(budget_s / max(1, runs + warmup) / max(t1, 1e-6)))))
    if nt_s > 1:
        ops.clear()  # free the calibration operators' buffers first
        ops = [build(nt_s, True)] + ([build(nt_s, False)] if forward_adjoint else [])
    for _ in range(warmup):
        apply_all(ops)
    times = [apply_all(ops) for _ in range(max(1, runs))]
    secs = float(np.median(times))
    upd = pts * nt_s * (2 if forward_adjoint else 1)
    what = "forward + adjoint operators" if forward_adjoint else "forward operator"
    sample = (f"reference {what} (acoustic_build + Operator::apply, JIT'd C/OpenMP, JIT "
              f"excluded) on {'x'.join(map(str, shape))} order {w.order}, {nt_s} of {w.nt} "
              f"time steps per apply, median of {len(times)} applies after {warmup} warm-up"
              + (f"; medium from the oracle's smooth-medium restatement ({t_med:.1f} s, "
                 "untimed)" if t_med is not None else "")
              + f"; OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')} "
              f"OMP_PLACES={os.environ.get('OMP_PLACES')}")
    # value = the median (the reference bench's protocol); best = the fastest
    # apply, the reference's own best case when other tenants load the host
    return {"value": upd / secs / 1e9, "unit": "GPts/s", "cores": threads, "kind": "reference",
            "sample": sample, "cpu": cpu_info(), "runs_s": times,
            "best": upd / min(times) / 1e9}


def ref_diffusion_sample(n, nt, budget_s, runs, warmup):
    _ref_threads()
    ol = _oracle()
    rng = np.random.default_rng(2016)
    u0 = np.zeros((n, n), np.float32)
    u0[1:-1, 1:-1] = rng.random((n - 2, n - 2))
    ref = ol.Ref()
    threads = ref.max_threads()
    ref.set_threads(threads)

    def build(k):
        op = ol.ref_diffusion(ref, n, n, (1, 2), (1, n - 1), k, 2)
        op.set("u", np.stack([u0, u0]))
        op.build()
        return op
    op = build(10)
    op.apply()
    t = time.perf_counter()
    op.apply()
    cal = (time.perf_counter() - t) / 10
    k = int(max(10, min(nt, budget_s / max(1, runs + warmup) / max(cal, 1e-9))))
    op = build(k)
    for _ in range(warmup):
        op.apply()
    times = []
    for _ in range(max(1, runs)):
        t = time.perf_counter()
        op.apply()
        times.append(time.perf_counter() - t)
    secs = float(np.median(times))
    return {"value": (n - 2) ** 2 * k / secs / 1e9, "unit": "GPts/s", "cores": threads,
            "kind": "reference", "cpu": cpu_info(), "runs_s": times,
            "best": (n - 2) ** 2 * k / min(times) / 1e9,
            "sample": f"reference diffusion operator on {n}^2, {k} of {nt} steps per apply, "
                      f"median of {len(times)} applies after {warmup} warm-up, JIT excluded"}


def config_block(w, parallelism):
    d = {"workload": f"{w.name}: 3D acoustic forward, space order {w.order}, "
                     f"{'x'.join(map(str, w.shape))} (boundary {w.bw}), {w.nt} time steps, "
                     f"dt {w.dt:.6g} s, {len(w.src_coords)} source(s), "
                     f"{len(w.rec_coords)} receivers",
         "grid": list(w.shape), "space_order": w.order, "nt": w.nt,
         "interior_points": interior_points(w.shape, w.order), "parallelism": parallelism,
         "bench_step": f"one full apply = {w.nt} time steps",
         "medium": ("two layers 1.5 / 2.5 km/s (build_medium)" if w.smooth is None else
                    f"seeded smooth random v in [1.5, 4.5] km/s: Gaussian-filtered hash noise, "
                    f"sigma {w.smooth['sigma']:g} cells, seed {w.smooth['seed']} "
                    "(csrc/medium.cu), sponge as build_medium"),
         "l2": "working set (3 u slots + m + eta) larger than the 126 MB L2; no flush needed"}
    return d


def diffusion_config_block(c):
    n, nt = c["n"], c["nt"]
    return {"workload": f"c1: 2D diffusion {n}^2, order 2, {nt} steps, alpha 1/2, "
                        f"dx 1/{n - 1}, dt = dx^2/4", "interior_points": (n - 2) ** 2,
            "bench_step": f"one full apply = {nt} time steps",
            "l2": "2 x 16 MiB slots are L2-resident (126 MB L2); HBM roofline is "
                  "a lower bound here"}


def ref_stable_dt():
    ol = _oracle()
    ref = ol.Ref()

    def f(order, vmax):
        return ref.lib.sfref_acoustic_stable_dt(3, np.array([64, 64, 64], np.int64), H, order,
                                                vmax, vmax)
    return f


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    c = CONFIGS[args.config]
    budget = args.ref_budget
    if c.get("kind") == "diffusion":
        base = ref_diffusion_sample(c["n"], c["nt"], budget, args.steps, args.warmup)
        pts = (c["n"] - 2) ** 2
        cfg = diffusion_config_block(c)
        ms = pts * c["nt"] / (base["value"] * 1e9) * 1e3
    else:
        w = workload(args.config, world, ref_stable_dt())
        fwi = c.get("kind") == "fwi"
        base = ref_acoustic_sample(w, budget, args.steps, args.warmup, forward_adjoint=fwi)
        pts = interior_points(w.block, w.order)
        cfg = config_block(w, f"reference CPU (one block of the {world}-GPU job)"
                           if world > 1 else "reference CPU")
        if fwi:
            cfg["workload"] = (f"c5: FWI forward + adjoint sweeps 301^3 order 8, {w.nt} steps "
                               "(the reference has no gradient: its two operators are timed)")
        ms = pts * w.nt * (2 if fwi else 1) / (base["value"] * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": "GPts/s (grid-point updates/sec)", "value": base["value"],
        "unit": "GPts/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": cfg,
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu")},
        "e2e": {"value": base["value"], "unit": "GPts/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    # the reference arm must not have touched the product (driver check)
    assert "paper_1609_03361_b200" not in sys.modules, "reference arm imported the product"
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arms

def product_stable_dt(sf):
    return lambda order, vmax: sf.api._stable_dt(3, order, H, vmax, vmax)


def roofline_line(ms_per_step, share, nt, pts, eta_skip, r, traffic):
    """Dominant kernel (the stencil): ALGORITHMIC bytes per launch -- SURVEY
    §8(d)'s compulsory 20 B per interior point (read u(t), u(t-1), m, eta;
    write u(t+1)) x the interior points of one launch -- over its average
    launch time inside the timed region. The kernel moves fewer bytes than
    that (all-zero eta boxes are never loaded): `moved_bytes_per_launch` and
    `frac_moved` report that stricter lens, `traffic` the ncu DRAM bytes."""
    stencil_launch_ms = ms_per_step / nt * share
    alg_bytes = 20.0 * pts
    moved = (20 - 4 * eta_skip) * pts
    peak, peak_kind = load_peaks()
    secs = stencil_launch_ms / 1e3
    achieved = alg_bytes / secs / 1e9
    ops = 21 + 13 * r
    return ({"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
             "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
             "kernel": f"3D stencil (radius {r}) avg launch {stencil_launch_ms * 1e3:.1f} us",
             "alg_bytes_per_launch": alg_bytes, "bytes_per_point": 20,
             "moved_bytes_per_launch": moved, "eta_boxes_skipped": eta_skip,
             "frac_moved": moved / secs / 1e9 / peak},
            # second lens for the high orders: the reference's exact fp32
            # operation count (no FMA contraction) against 148 SMs x 128 lanes
            {"bound": "fp32", "ops_per_point": ops,
             "achieved": ops * pts / secs / 1e12,
             "peak": 148 * 128 * 1.965e9 / 1e12, "unit": "Tops/s",
             "frac": ops * pts / secs / (148 * 128 * 1.965e9),
             "peak_source": "148 SMs x 128 fp32 lanes x 1965 MHz (max SM clock)"})


def traffic_of(key):
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(tpath)).get(key)
    except Exception:
        return None


def b200_setup(sf, w, device=0, pinned=False, nt=None):
    """The config's forward operator through the mirrored reference API
    (acoustic_build), its medium generated on the GPU for smooth configs."""
    model = sf.AcousticModel(shape=w.shape, boundary_width=w.bw, spacing=w.h,
                             nt=w.nt if nt is None else nt, dt=w.dt, space_order=w.order,
                             f0=w.f0, v_top=w.v_top, v_bottom=w.v_bottom,
                             src_coords=w.src_coords, rec_coords=w.rec_coords)
    smooth = None
    if w.smooth is not None:
        smooth = sf.SmoothMedium(shape=w.shape, seed=w.smooth["seed"], sigma=w.smooth["sigma"],
                                 v_lo=w.smooth["v_lo"], v_hi=w.smooth["v_hi"],
                                 boundary_width=w.bw, spacing=w.h, v_min=w.smooth["v_min"])
    return sf.acoustic_build(model, True, device=device, pinned=pinned, smooth=smooth)


def run_b200_arm(args, local):
    import torch

    import paper_1609_03361_b200 as sf
    w = workload(args.config, 1, product_stable_dt(sf))
    setup = b200_setup(sf, w, device=local, pinned=True)
    op = setup.op
    pts = interior_points(w.shape, w.order)
    r = w.order // 2
    # resident: upload once, warm up (graph capture + clocks), then time
    op.upload()
    for _ in range(args.warmup):
        op.run(0, w.nt)
    op.synchronize()
    torch.cuda.set_device(local)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        total = 0.0
        nl = 0
        for _ in range(args.steps):
            t, _, nl = op.time(stencil=False)
            total += t
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    ms_per_step = total / args.steps
    value = pts * w.nt / (ms_per_step / 1e3) / 1e9
    # the stencil's share of a run: a full run and a stencil-only run timed
    # back to back right after the timed region (same power / clock state)
    tot2, sten2, _ = op.time(stencil=True)
    share = min(1.0, sten2 / tot2) if tot2 > 0 else 1.0
    roof, comp = roofline_line(ms_per_step, share, w.nt, pts, op.eta_skip_fraction(), r,
                               traffic_of(args.config))
    # e2e through the C-ABI apply with pinned host buffers
    h2d = sum(a.data.nbytes for a in op.args)
    d2h = setup.field.data.nbytes + setup.rec.data.data.nbytes
    op.apply()  # warm
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.apply()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e = pts * w.nt / e2e_s / 1e9
    del setup, op
    base = None
    if not args.no_cpu_baseline:
        try:
            base = ref_acoustic_sample(w, args.cpu_budget, 3, 1)
        except Exception as e:  # reported, not fatal
            base = {"error": str(e)}
    line = {
        "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "ms_per_time_step": ms_per_step / w.nt,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_block(w, "single GPU"),
        "roofline": roof, "compute_roofline": comp, "stencil_share": share,
        "cpu_baseline": base,
        "e2e": {"value": e2e, "unit": "GPts/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(nl * args.steps), "clocks": clocks.summary(),
        "wall_s_timed_region": t_wall,
    }
    print(json.dumps(line), flush=True)


def run_b200_diffusion(args, local):
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
    # work per apply is identical)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.apply()
    e2e_s = (time.perf_counter() - t0) / args.steps
    base = None
    if not args.no_cpu_baseline:
        base = ref_diffusion_sample(n, nt, args.cpu_budget, 3, 1)
    l2 = traffic_of("c1")
    line = {
        "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "ms_per_time_step": ms / nt,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": diffusion_config_block(c),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": l2, "peak_source": peak_kind,
                     "kernel": f"diffusion_tb_kernel (temporal blocking, T=8 steps per "
                               f"launch), {launch_ms * 1e3:.2f} us per time step",
                     "alg_bytes_per_launch": 8 * pts,
                     "note": "achieved = 8 B/pt per time step over the time per step; the "
                             "field is L2-resident, so HBM does not bind: `traffic` is the "
                             "L2 / shared-memory lens of the kernel (ncu, profiles/"
                             "r2_ncu_kernels.txt r2_tb_c1)"},
        "cpu_baseline": base,
        "e2e": {"value": pts * nt / e2e_s / 1e9, "unit": "GPts/s",
                "h2d_bytes_per_step": b.u.data.nbytes, "d2h_bytes_per_step": b.u.data.nbytes},
        "gpu_launches": int(nl * args.steps), "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_b200_fwi(args, local):
    """C5: forward with the full wavefield history in HBM (nt+2 levels of
    301^3), adjoint injecting seeded N(0,1) residuals at 201 x 201 surface
    receivers, gradient accumulated in the adjoint stencil. The metric counts
    the updates of both passes."""
    import paper_1609_03361_b200 as sf
    c = CONFIGS[args.config]
    shape, order, nt = tuple(c["shape"]), c["order"], c["nt"]
    r = order // 2
    dt = min(0.4 * H / 4500.0, sf.api._stable_dt(3, order, H, 4500.0, 4500.0))
    sm = sf.SmoothMedium(shape=shape, boundary_width=BW, spacing=H, **{
        k: v for k, v in SMOOTH.items()})
    lo, hi = sm.extrema(device=local)
    m, eta = sm.generate(lo, hi, device=local)
    mid = shape[1] // 2
    src_c = [[(BW + 2) * H, mid * H, mid * H]]
    rec_c = [[(BW + 10) * H, (BW + i) * H, (BW + j) * H] for i in range(201) for j in range(201)]

    def interp(coords):
        cis, ws = zip(*[sf.interpolation_weights(cc, H, shape) for cc in coords])
        return np.array(cis, np.int32), np.array(ws, np.float32)
    src_ci, src_w = interp(src_c)
    rec_ci, rec_w = interp(rec_c)
    t0 = 1.0 / 10.0
    src = np.array([sf.ricker_wavelet(10.0, t * dt, t0) for t in range(nt)], np.float32)[:, None]
    rng = np.random.default_rng(5)
    residual = rng.standard_normal((nt, len(rec_c)), dtype=np.float32)
    plan = sf.FwiPlan(shape, order, nt, dt, H, 1, len(rec_c), device=local, pinned=True)
    # inputs resident in page-locked host memory, outputs into the plan's
    # page-locked buffers: the copies inside the timed call run at the PCIe rate
    m, eta, residual, src = (sf.api.pinned_array(x.shape, np.float32, like=x)
                             for x in (m, eta, residual, src))
    # warm-up call (graph capture, sparse index build), then the timed one
    plan.gradient(m, eta, src, src_ci, src_w, rec_ci, rec_w, residual)
    t_e = time.perf_counter()
    rec_out, grad, _, _ = plan.gradient(m, eta, src, src_ci, src_w, rec_ci, rec_w, residual)
    e2e_s = time.perf_counter() - t_e
    fwd = adj = 0.0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            f, a = plan.time()
            fwd += f
            adj += a
    fwd /= args.steps
    adj /= args.steps
    pts = interior_points(shape, order)
    value = 2 * pts * nt / ((fwd + adj) / 1e3) / 1e9
    peak, peak_kind = load_peaks()
    skip = plan.eta_skip_fraction()
    # SURVEY 8(d)'s algorithmic bytes per point: forward 20 B, adjoint +
    # gradient 36 B (the all-zero eta boxes the kernels skip are not
    # subtracted; `moved_frac` is that stricter lens)
    bf, ba = 20.0, 36.0
    mf, ma = 20 - 4 * skip, 36 - 4 * skip
    base = None
    if not args.no_cpu_baseline:
        try:
            w = SimpleNamespace(name="c5", block=shape, shape=shape, order=order, nt=nt, bw=BW,
                                h=H, f0=10.0, dt=dt, v_top=4500.0, v_bottom=4500.0,
                                smooth=dict(SMOOTH, shape=shape), src_coords=src_c,
                                rec_coords=rec_c)
            base = ref_acoustic_sample(w, args.cpu_budget, 3, 1, forward_adjoint=True)
        except Exception as e:
            base = {"error": str(e)}
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
                     "moved_frac": (mf + ma) * pts * nt / ((fwd + adj) / 1e3) / 1e9 / peak,
                     "traffic": traffic_of("c5"), "eta_boxes_skipped": skip},
        "cpu_baseline": base,
        "e2e": {"value": 2 * pts * nt / e2e_s / 1e9, "unit": "GPts/s",
                "h2d_bytes_per_step": m.nbytes * 2 + residual.nbytes + src.nbytes,
                "d2h_bytes_per_step": grad.nbytes + rec_out.nbytes},
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_b200_slabs(args, world, rank, local):
    """N > 1 (or --force-slabs): weak scaling over depth slabs. The global grid
    stacks one config block per GPU along axis 0; rank g owns one block's
    planes and swaps r-deep halos with its neighbours over NCCL inside every
    time step (sf_plan_attach_nccl). Smooth media are generated per slab on
    the rank's GPU from global indices, with the global extrema reduced over
    ranks; no rank ever holds the global medium."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200 import _lib
    from paper_1609_03361_b200.slab import SlabPartition, SlabRun, nccl_unique_id
    w = workload(args.config, world, product_stable_dt(sf))
    gshape = w.shape
    r = w.order // 2
    part = SlabPartition.split(gshape[0], r, world, rank)
    lshape = (part.local_n0,) + tuple(gshape[1:])
    if w.smooth is None:
        model = sf.AcousticModel(shape=gshape, boundary_width=w.bw, spacing=w.h, nt=w.nt,
                                 dt=w.dt, space_order=w.order, f0=w.f0, v_top=w.v_top,
                                 v_bottom=w.v_bottom)
        m, eta = sf.build_medium(sf.Grid(), model)
        m_loc = np.ascontiguousarray(m.data[part.local()])
        eta_loc = np.ascontiguousarray(eta.data[part.local()])
    else:
        sm = sf.SmoothMedium(shape=gshape, seed=w.smooth["seed"], sigma=w.smooth["sigma"],
                             v_lo=w.smooth["v_lo"], v_hi=w.smooth["v_hi"], boundary_width=w.bw,
                             spacing=w.h, v_min=w.smooth["v_min"])
        lo, hi = sm.extrema(part.own_begin, part.own_end, device=local)
        lo = reduce_over_ranks(world, lo, "min")
        hi = reduce_over_ranks(world, hi, "max")
        m_loc, eta_loc = sm.generate(lo, hi, part.plane0, part.plane_end, device=local)

    def interp(coords):
        cis, ws = zip(*[sf.interpolation_weights(cc, w.h, gshape) for cc in coords])
        return np.array(cis, np.int32), np.array(ws, np.float32)
    src_ci, src_w = interp(w.src_coords)
    rec_ci, rec_w = interp(w.rec_coords)
    t0 = 1.0 / w.f0
    ser = np.array([sf.ricker_wavelet(w.f0, t * w.dt, t0) for t in range(w.nt)],
                   np.float32)[:, None].repeat(len(src_ci), axis=1)
    rec = np.zeros((w.nt, len(rec_ci)), np.float32)
    slab = SlabRun(part, gshape, w.order, True, w.nt, w.dt, w.h, m_loc, eta_loc, ser, src_ci,
                   src_w, rec, rec_ci, rec_w, device=local, local_medium=True)
    del m_loc, eta_loc
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    with stdout_to_stderr():
        slab.attach_nccl(obj[0], world, rank)
    for _ in range(args.warmup):
        slab.run(0, w.nt)
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
    ms_per_step = reduce_over_ranks(world, total / args.steps)
    # per-rank stencil-only pass (no exchange) for the roofline of the kernel
    sf.api.check(_lib.lib.sf_plan_time(slab.plan, C.byref(tot), C.byref(sten), C.byref(nl)))
    share = reduce_over_ranks(world, min(1.0, sten.value / tot.value) if tot.value > 0 else 1.0)
    pts = interior_points(gshape, w.order)
    value = pts * w.nt / (ms_per_step / 1e3) / 1e9
    frac = C.c_double()
    sf.api.check(_lib.lib.sf_plan_eta_skip_fraction(slab.plan, C.byref(frac)))
    own_pts = interior_points(w.block, w.order)  # a rank's share of the interior
    roof, comp = roofline_line(ms_per_step, share, w.nt, own_pts, frac.value, r, None)
    # e2e: upload host slices, run, download, every step (pinned host buffers,
    # as in the single-GPU arm)

    def pinned(a):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        arr = t.numpy()
        arr[...] = a
        return arr, t
    # every rank of the node pins its own slab's nine arrays at once: check
    # the host has room (a rank replaces its pageable arrays one at a time)
    need = float(sum(b.nbytes for b in slab.bufs))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    try:
        import psutil
        avail = float(psutil.virtual_memory().available)
    except Exception:
        avail = float("inf")
    room = reduce_over_ranks(world, 1.0 if 1.3 * need * local_world < avail else 0.0, "min")
    e2e = None
    if room > 0:
        keep = []
        for i in range(len(slab.bufs)):
            arr, t = pinned(slab.bufs[i])
            slab.bufs[i] = arr
            keep.append(t)
        barrier(world)
        t_e = time.perf_counter()
        for _ in range(args.steps):
            argv = (C.c_void_p * 9)(*[b.ctypes.data for b in slab.bufs])
            sf.api.check(_lib.lib.sf_plan_invoke(slab.plan, argv, 9))
        e2e_s = reduce_over_ranks(world, (time.perf_counter() - t_e) / args.steps)
        h2d = reduce_over_ranks(world, float(sum(b.nbytes for b in slab.bufs))) * world
        d2h = reduce_over_ranks(world, float(slab.bufs[0].nbytes + slab.bufs[6].nbytes)) * world
        e2e = {"value": pts * w.nt / e2e_s / 1e9, "unit": "GPts/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
    else:
        e2e = {"value": None, "unit": "GPts/s",
               "skipped": f"host memory: {local_world} ranks x {need / 1e9:.1f} GB pinned "
                          f"exceeds the {avail / 1e9:.0f} GB available"}
    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            base = ref_acoustic_sample(w, args.cpu_budget, 3, 1)
        except Exception as e:
            base = {"error": str(e)}
    if rank == 0:
        cfg = config_block(w, f"slab{world}")
        cfg["workload"] += (f"; {world} depth slab(s) of {w.block[0]} planes, NCCL halo "
                            f"exchange ({r} planes per face) every step")
        cfg["local_grid"] = list(lshape)
        line = {
            "metric": "GPts/s (grid-point updates/sec)", "value": value, "unit": "GPts/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "ms_per_time_step": ms_per_step / w.nt,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": cfg, "roofline": roof, "compute_roofline": comp,
            "stencil_share": share, "cpu_baseline": base,
            "e2e": e2e,
            "gpu_launches": int(nl.value * args.steps),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    slab.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of CPU work for the product line's cpu_baseline sample")
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="seconds of CPU work for the reference arm's timed applies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # exercise the multi-GPU slab path (NCCL communicator, slab plans) with a
    # single rank: validates the N > 1 code on a one-GPU box
    ap.add_argument("--force-slabs", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_init()
    if rank != 0:  # only rank 0 writes stdout (its one JSON line)
        sys.stdout.flush()
        os.dup2(2, 1)
    kind = CONFIGS[args.config].get("kind", "acoustic")
    if args.impl == "reference":
        # rank 0 alone runs the CPU reference; the others exit without work
        run_reference_arm(args, world, rank)
        return
    if world > 1:
        with stdout_to_stderr():
            dist_start(local)
    try:
        if kind == "diffusion":
            if rank == 0:
                run_b200_diffusion(args, local)
        elif kind == "fwi":
            if rank == 0:
                run_b200_fwi(args, local)
        elif world > 1 or args.force_slabs:
            run_b200_slabs(args, world, rank, local)
        else:
            run_b200_arm(args, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
