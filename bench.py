#!/usr/bin/env python
"""Benchmark: particle-updates/s of the short-range gravity + CRK-SPH force
evaluation (BASELINE.json metric), on synthetic Zel'dovich-displaced
two-species lattices.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cX] [--impl ours|reference]

Default workload: c2 (2x128^3, configs[1]) at N = 1; c4 (2x512^3, configs[3], the
multi-GPU config BASELINE.json names) at N > 1.  c3 (clustered) and c5
(gravity-only 1024^3 DM, >= 4 GPUs) run with --config.

A step is one force evaluation at depth 0: bin sort + k-d leaf
build + reorder, leaf-pair lists, one neighbour-count pass, density + EOS, CRK
moments + 3x3 solve, short-range gravity, hydro force.  ``value`` times
hb_force_step on device-resident inputs (CUDA events, max over ranks);
``e2e`` times the same through host buffers (pinned H2D of the particle fields,
the step, D2H of the results).  ``--impl reference`` times the reference
algorithm's CPU restatement (oracle/, pinned bitwise to the reference) on the
host cores: there is no other CPU implementation that can travel to the box.
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

METRIC = "particle-updates/sec (short-range grav+CRK-SPH) at 1/2/4/8 B200; % FP32 peak"
UNIT = "particle-updates/s"
# reference OpCost per in-support ordered pair (FMA = 2): hb/kernels.py:523,544,555,567,601
OPCOST = {"gravity": 29, "density": 16, "ncount": 7, "crk": 29, "hydro": 57}

CONFIGS = {
    # name: (npd, sigma_psi in lattice spacings, species, description)
    "c1": (32, 0.05, "both", "2x32^3 particles (DM + baryon), one short-range gravity + CRK-SPH step"),
    "c2": (128, 0.05, "both", "2x128^3 particles, z=10 near-uniform Zel'dovich ICs, single B200"),
    "c3": (256, 2.0, "both", "2x256^3 particles, z=0 strongly clustered (neighbour-count imbalance)"),
    "c4": (512, 0.05, "both", "2x512^3 particles, spatial decomposition with ghost exchange "
                              "at 2/4/8 B200"),
    "c5": (1024, 0.05, "dm", "gravity-only 1024^3 dark-matter particles, short-range PP kernel "
                             "sweep (>= 4 B200)"),
}
DEVICE_IC_ABOVE = 1 << 29   # particles: displacement field built on the GPU (numpy: ~60 GB/rank)
# default workload per GPU count: configs[1] at N = 1 (the metric's single-GPU
# config), configs[3] -- the config BASELINE.json names for 2/4/8 GPUs and its
# strong-scaling target -- at N > 1
DEFAULT_CONFIG = {1: "c2"}
DEFAULT_CONFIG_MULTI = "c4"
SUBBOX_ABOVE = 40_000_000   # CPU samples above this size use an interior sub-box


def peaks():
    """FP32 roofline denominator: FFMA peak measured on this pool's B200
    (profiles/peaks_r01.json; MEASURED_PEAKS.json carries no FP32 entry)."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "peaks_r01.json")))
        return float(rec["ffma_reg_tflops"]), "measured FFMA (profiles/peaks_r01.json)"
    except Exception:
        return 148 * 128 * 2 * 1.965e9 / 1e12, "nominal 148 SM x 128 lanes x 2 x 1.965 GHz"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = int(gpu)
        self.proc = None
        self.lines = []
        self.window = None

    def start(self):
        """Begin sampling (before warm-up, so nvidia-smi is running when the
        timed window opens); mark the window with begin() / end()."""
        return self.__enter__()

    def begin(self):
        self.window = [time.time(), None]

    def end(self):
        self.window[1] = time.time()
        # wait (<= 5 s) for a sample stamped after the window: it bounds the
        # window from above and flushes the pipe's buffered lines
        t_stop = time.time() + 5.0
        while time.time() < t_stop and not any(
                (self._stamp(ln) or 0) > self.window[1] for ln in self.lines[-3:]):
            time.sleep(0.05)
        self.__exit__()

    @staticmethod
    def _stamp(ln):
        try:
            from datetime import datetime
            return datetime.strptime(ln.split(",")[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except Exception:
            return None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
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

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None and self.window[1] is not None:
            # samples inside the timed window, plus the nearest one on each side
            # (a window shorter than the 100 ms period may hold none)
            t0, t1 = self.window
            st = [(self._stamp(ln), ln) for ln in self.lines]
            st = [(t, ln) for t, ln in st if t is not None]
            inside = [ln for t, ln in st if t0 <= t <= t1]
            before = [ln for t, ln in st if t < t0][-1:]
            after = [ln for t, ln in st if t > t1][:1]
            lines = before + inside + after
        for ln in lines:
            parts = [x.strip() for x in ln.split(",")][1:]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(cfg_name: str, rank: int = 0, world: int = 1, local: bool = False,
                  region=None):
    """Synthetic workload; local=True (world > 1) materialises only the rows
    rank `rank` owns (identical to selecting them from the full set), so the
    host never holds world copies of a 2x512^3 set; region = (lo, hi) keeps
    only the particles inside that cube (the reference arm's sub-box sample).
    Above DEVICE_IC_ABOVE particles the displacement field is built on the
    GPU (ic.make_zeldovich_ic_device) and a selection is required."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.distributed import rank_grid_for
    from paper_2510_03557_b200.domain import owner_ranks, owner_ranks_torch
    from paper_2510_03557_b200.ic import make_zeldovich_ic, make_zeldovich_ic_device
    from paper_2510_03557_b200.resident import StepConfig
    npd, sigma, species, desc = CONFIGS[cfg_name]
    box = BoxGeometry(1.0)
    n_all = (2 if species == "both" else 1) * npd ** 3
    on_device = n_all > DEVICE_IC_ABOVE
    select = None
    if region is not None:
        rlo, rhi = (float(v) for v in region)
        if on_device:
            select = lambda pos: ((pos >= rlo) & (pos < rhi)).all(dim=1)  # noqa: E731
        else:
            select = lambda pos: np.all((pos >= rlo) & (pos < rhi), axis=1)  # noqa: E731
    elif local and world > 1:
        grid = rank_grid_for(world)
        if on_device:
            select = lambda pos: owner_ranks_torch(pos, box, grid) == rank  # noqa: E731
        else:
            select = lambda pos: owner_ranks(pos, box, grid) == rank  # noqa: E731
    if on_device:
        if select is None:
            raise ValueError(f"{cfg_name} is built per rank or per region only (--gpus >= 4)")
        p = make_zeldovich_ic_device(npd, box, sigma, select, species=species)
    else:
        p = make_zeldovich_ic(npd, box, sigma, species=species, select=select)
    d = 1.0 / npd
    pm_grid = 2 * npd                       # pm_grid_n = 2 npd
    pm_cell = 1.0 / pm_grid
    r_s = 2.0 * pm_cell                     # hb/config.py:87-90
    r_cut = 5.0 * r_s                       # hb/config.py:91-93
    eps = (1.0 / n_all ** (1.0 / 3.0)) / 50.0  # hb/config.py:95-99
    h_max = 1.3 * d if species == "both" else 0.0   # gas smoothing of the IC
    reach = max(r_cut, 2.0 * h_max)
    bin_width = max(4.0 * pm_cell, reach * (1 + 1e-9))  # hb/driver.py:147-150
    cfg = StepConfig(box=box, bin_width=bin_width, max_leaf_size=256, r_s=r_s, r_cut=r_cut,
                     softening=eps)
    meta = {"workload": desc, "config": cfg_name, "n_particles": n_all,
            "n_gas": npd ** 3 if species == "both" else 0,
            "n_per_dim": npd, "sigma_psi_spacings": sigma,
            "smoothing": "h = 1.3 d (unadapted)" if species == "both" else "none (gravity only)",
            "passes": "all" if species == "both" else "gravity",
            "ic_fft": "cuFFT (GPU)" if on_device else "numpy",
            "r_s": "d", "r_cut": "5 d", "softening": "L/N^(1/3)/50", "max_leaf_size": 256,
            "mesh": "bare periodic box, bin width max(4 PM cells, reach)",
            "bins_per_axis": int(np.floor(1.0 / bin_width)),
            "ic": "Zel'dovich, seed 2510035570, P(k)~k^-2 exp(-(kd)^2)",
            "l2": "working set > 126 MB L2 (no flush needed)"}
    return p, cfg, meta


def pair_counts(p, cfg):
    """Exact in-support ordered pair counts for the algorithmic-FLOP roofline
    (untimed; uses the compat API's exact pairs_in_reach)."""
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.kernels import counting_kernel, neighbor_count_kernel
    from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
    q = p.copy()
    mesh = build_mesh_and_leaves(q, cfg.box, cfg.bin_width, cfg.max_leaf_size)
    reach = max(cfg.r_cut, 2 * float(q.smoothing.max()))
    il = assemble_interaction_lists(mesh, reach, 0)
    st = q.state_matrix(cfg.eos_gamma)
    g = eval_interaction_list(counting_kernel(cfg.r_cut), il, st, mesh, mode=EvalMode.RELAXED)
    nc = eval_interaction_list(neighbor_count_kernel(2 * float(q.smoothing.max())), il, st, mesh,
                               mode=EvalMode.DETERMINISTIC)
    gas = q.species == 1
    sph_in = int(nc.values[gas, 0].sum())          # r <= 2 h_i, gas-gas, incl. self
    n_gas = int(gas.sum())
    return {"gravity": int(g.values[:, 0].sum()), "density": sph_in, "ncount": sph_in,
            "crk": sph_in, "hydro": sph_in - n_gas,
            "gravity_scheduled_leafpairs": int(g.counters["pairs_scheduled"])}


def subbox_region(L: float, r_cut: float, n_all: int, h_max: float,
                  n_target: int = 2 * 128 ** 3):
    """(a, side, reach) of the interior sample cube [a, a + side)^3 holding
    ~n_target of n_all particles; its shell reaches `reach` further out."""
    side = L * min(1.0, (n_target / n_all) ** (1.0 / 3.0))
    return 0.5 * (L - side), side, max(r_cut, 2 * h_max)


def subbox_sample(p, cfg, n_target: int = 2 * 128 ** 3, n_all: int | None = None):
    """Interior cube of the workload holding ~n_target owned particles plus its
    overload shell (width = reach) as ghosts, on a bounded mesh -- the domain
    one rank of a spatial decomposition sees.  Returns (ParticleSet, bounds_lo,
    bounds_hi).  Per-particle work matches the full box (same lattice
    statistics), so owned / time is the full workload's rate.  p may already
    be restricted to the shell's outer cube (then pass the full n_all)."""
    a, side, reach = subbox_region(cfg.box.side_length, cfg.r_cut, n_all or p.n,
                                   float(p.smoothing.max()), n_target)
    x = p.pos
    inner = np.all((x >= a) & (x < a + side), axis=1)
    shell = np.all((x >= a - reach) & (x < a + side + reach), axis=1) & ~inner
    idx = np.concatenate([np.nonzero(inner)[0], np.nonzero(shell)[0]])
    q = p.select(idx)
    q.ghost[:] = 0
    q.ghost[int(inner.sum()):] = 1
    q.image_shift[:] = 0
    lo = np.full(3, a - reach)
    hi = np.full(3, a + side + reach)
    return q, lo, hi


def cpu_baseline(p, cfg, frac: float = 1 / 32, threads: int | None = None, bounds=None,
                 gravity_only: bool = False):
    """The reference algorithm (oracle/ C restatement, bitwise-pinned to the
    reference) on the host cores: full build + lists, every (1/frac)-th entry
    of each kernel's list scaled up (fixed per-call cost measured separately),
    full CRK solve.  Gravity and hydro use the reference driver's mirror mode
    over unordered pairs (half the pair work).  bounds: (lo, hi) of a bounded
    (rank-domain) mesh, else the periodic box."""
    from oracle import oracle as O
    from paper_2510_03557_b200.kernels import (crk_moments_kernel, density_kernel,
                                               hydro_force_kernel, neighbor_count_kernel)
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    threads = threads or os.cpu_count() or 1
    O.set_threads(threads)
    L = cfg.box.side_length
    t0 = time.perf_counter()
    blo, bhi = bounds if bounds is not None else (None, None)
    m = O.build_mesh(p.pos, p.image_shift, p.ghost, L, cfg.bin_width, cfg.max_leaf_size,
                     bounds_lo=blo, bounds_hi=bhi)
    t_build = time.perf_counter() - t0
    h_max = float(p.smoothing.max())
    reach = max(cfg.r_cut, 2 * h_max)
    t0 = time.perf_counter()
    la, lb, ls = O.assemble(m, L, reach)
    t_list = time.perf_counter() - t0
    perm = m["perm"]
    st = O.state_matrix(p.pos[perm], p.vel[perm], p.mass[perm], p.smoothing[perm],
                        p.density[perm], p.internal_energy[perm], p.species[perm], cfg.eos_gamma)
    ua, ub, us, _ = O.unordered_due_pairs(la, lb, ls, m["leaf_start"].shape[0])
    gk = short_range_gravity_kernel(ForceSplit(r_s=cfg.r_s, r_cut=cfg.r_cut), cfg.softening)
    jobs = [("ncount", neighbor_count_kernel(2 * h_max), False),
            ("density", density_kernel(2 * h_max), False),
            ("crk", crk_moments_kernel(2 * h_max), False),
            ("gravity", gk, True),
            ("hydro", hydro_force_kernel(2 * h_max), True)]
    if gravity_only:   # the gravity-only configs' step: build + lists + gravity
        jobs = [j for j in jobs if j[0] == "gravity"]
    times = {}
    for name, ker, mirror in jobs:
        A, B, S = (ua, ub, us) if mirror else (la, lb, ls)
        # every stride-th entry: the sample spans the whole list (per-entry
        # cost varies along it, so a leading slice extrapolates poorly)
        stride = max(1, int(round(1.0 / frac)))
        As, Bs, Ss = A[::stride], B[::stride], S[::stride]
        k = max(1, len(As))
        mode = "deterministic" if name == "ncount" else "relaxed"
        t0 = time.perf_counter()
        O.eval_pairs(ker, A[:0], B[:0], S[:0], st, m["leaf_start"], m["leaf_end"], L, mode=mode,
                     workers=threads, mirror=mirror)
        t_fixed = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.eval_pairs(ker, As, Bs, Ss, st, m["leaf_start"], m["leaf_end"], L, mode=mode,
                     workers=threads, mirror=mirror)
        t_s = time.perf_counter() - t0
        times[name] = t_fixed + max(t_s - t_fixed, 0.0) * len(A) / k
    if not gravity_only:
        t0 = time.perf_counter()
        vals = np.zeros((p.n, 10))
        vals[:, 0] = 1.0
        vals[:, 4] = vals[:, 7] = vals[:, 9] = 1.0
        O.crk_solve(vals, p.species[perm] == 1)
        times["crk_solve"] = time.perf_counter() - t0
    total = t_build + t_list + sum(times.values())
    n_owned = int(np.count_nonzero(p.ghost == 0))
    return {"value": n_owned / total, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"full build+lists ({t_build:.2f}+{t_list:.2f} s), every "
                       f"{max(1, int(round(1.0 / frac)))}th entry of each "
                       f"kernel's list (ordered: ncount/density/crk; mirror-unordered: "
                       f"gravity/hydro) scaled to the full list, full CRK solve; "
                       f"est. step {total:.1f} s"),
            "seconds": {"build": t_build, "list": t_list, **times, "total_est": total}}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    npd, _, species, _ = CONFIGS[args.config]
    n_all = (2 if species == "both" else 1) * npd ** 3
    bounds, where = None, ""
    if n_all > SUBBOX_ABOVE:   # build only the sample cube and its shell
        h = 1.3 * (1.0 / npd) if species == "both" else 0.0
        a, side, reach = subbox_region(1.0, 5.0 / npd, n_all, h)   # r_cut = 5 d (make_workload)
        p, cfg, meta = make_workload(args.config, region=(a - reach, a + side + reach))
        p, lo, hi = subbox_sample(p, cfg, n_all=n_all)
        bounds = (lo, hi)
        where = (f"interior sub-box of {int(np.count_nonzero(p.ghost == 0))} owned + "
                 f"{int(np.count_nonzero(p.ghost))} overload-shell particles (bounded mesh); ")
    else:
        p, cfg, meta = make_workload(args.config)
    vals = []
    base = None
    gonly = species == "dm"
    for _ in range(args.warmup):
        cpu_baseline(p, cfg, frac=args.cpu_frac / 4, bounds=bounds, gravity_only=gonly)
    for _ in range(args.steps):
        base = cpu_baseline(p, cfg, frac=args.cpu_frac, bounds=bounds, gravity_only=gonly)
        vals.append(base["value"])
    v = float(np.median(vals))
    n_owned = meta["n_particles"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": n_owned / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": meta,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": "port",
                             "sample": where + base["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _make_rank(args, p, cfg, rank, world, meta, group=None, local=False):
    """N = 1: the bare periodic mesh; N > 1: cuboid rank + overload exchange.
    local: p already holds only this rank's rows."""
    from paper_2510_03557_b200.distributed import DistributedRank, rank_grid_for
    from paper_2510_03557_b200.domain import owner_ranks
    from paper_2510_03557_b200.resident import PASS_ALL, PASS_GRAVITY, ResidentRank
    if world == 1:
        return ResidentRank(p, cfg, gravity_only=meta["n_gas"] == 0)
    if not local:
        owner = owner_ranks(p.pos, cfg.box, rank_grid_for(world))
        p = p.select(np.nonzero(owner == rank)[0])
    gas = meta["n_gas"] > 0
    h = 1.3 * (1.0 / CONFIGS[meta["config"]][0]) if gas else 0.0   # IC gas smoothing (ic.py)
    return DistributedRank(p, cfg.box, rank, world, cfg.r_s, cfg.r_cut, cfg.softening, h, h,
                           cfg.max_leaf_size, group=group, n_global=meta["n_particles"],
                           passes=PASS_ALL if gas else PASS_GRAVITY)


def run_gpu_arm(args):
    import torch
    from paper_2510_03557_b200 import _native as N
    from paper_2510_03557_b200.resident import PASS_ALL, PASS_GRAVITY, STEP_FIELDS
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    npd_c, _, species_c, _ = CONFIGS[args.config]
    passes = PASS_ALL if species_c == "both" else PASS_GRAVITY
    rank_rows = world > 1 and npd_c ** 3 * (2 if species_c == "both" else 1) > SUBBOX_ABOVE
    p, cfg, meta = make_workload(args.config, rank, world, local=rank_rows)
    n_total = meta["n_particles"]
    rr = _make_rank(args, p, cfg, rank, world, meta, local=rank_rows)
    engine = rr if world == 1 else None
    lib = N.lib()
    stream = torch.cuda.current_stream()

    def step(timing=False):
        if world == 1:
            rr.step(passes, timing=timing)
            return rr.last
        rr.step(timing=timing)
        return rr.engine.last

    clocks = ClockSampler(local).start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    l0 = lib.hb_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases = []
    torch.cuda.synchronize()
    clocks.begin()
    ev0.record(stream)
    for _ in range(args.steps):
        phases.append(step(timing=True)["ms_phase"])
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks.end()
    launches = lib.hb_launch_count() - l0
    ms_total = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = n_total / (ms_step * 1e-3)
    ph = {k: float(np.mean([x[k] for x in phases])) for k in phases[0]}
    if dist:
        t = torch.tensor([ph["gravity"], ph["k_gravity"]], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ph["gravity_max_over_ranks"] = float(t[0].item())
        ph["k_gravity_max_over_ranks"] = float(t[1].item())

    # ---- e2e: pinned host inputs -> device -> step (exchange incl.) -> results to host;
    # each call's copies overlap only that call's own compute (HostStepper)
    if world == 1:
        src_fields = {f: getattr(p, f) for f in STEP_FIELDS}
    else:
        own = rr.owned_fields["ghost"] == 0  # the rank set's owned rows are the host inputs
        src_fields = {f: rr.owned_fields[f][own].cpu().numpy() for f in STEP_FIELDS}
    pinned_in = {f: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                 for f, a in src_fields.items()}
    eng = rr if world == 1 else rr.engine
    out_names = (("grav", "hydro", "ncount", "crk_A", "crk_B", "perm") if passes == PASS_ALL
                 else ("grav", "perm"))
    pinned_out = {k: torch.empty(eng.out[k].shape, dtype=eng.out[k].dtype).pin_memory()
                  for k in out_names}
    if passes == PASS_ALL:
        pinned_out["density"] = torch.empty(eng.n, dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in pinned_in.values())
    d2h = sum(t.numel() * t.element_size() for t in pinned_out.values())

    # N > 1: the owned rows land in the engine's reorder buffer, free between
    # steps (the exchange reads them into the rank set before the step
    # overwrites it) -- no second copy of the rank's fields on the device
    e2e_dev = None if world == 1 else {
        f: rr.engine._buf1_store[f][:pinned_in[f].shape[0]] for f in STEP_FIELDS}

    host_stepper = None
    if world == 1:
        from paper_2510_03557_b200.resident import HostStepper
        host_stepper = HostStepper(rr, pinned_in, pinned_out, passes)
    else:
        # rank set: the exchange reads every input field, so the H2D copies
        # precede it; the SPH outputs, density and permutation drain while
        # gravity runs (sph_done), the gravity output after; deferred status
        s_out = torch.cuda.Stream()
        ev_sph, ev_done, ev_gh = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
        for ev in (ev_sph, ev_done, ev_gh):
            ev.record()
        status = torch.zeros(3, dtype=torch.int64, pin_memory=True)

    def e2e_step():
        if host_stepper is not None:
            host_stepper()
            return
        dst = rr.owned_fields = e2e_dev
        for f in STEP_FIELDS:
            dst[f].copy_(pinned_in[f], non_blocking=True)
        status.zero_()
        rr.step(sph_done=ev_sph, status=status, grav_half=ev_gh)
        main = torch.cuda.current_stream()
        ev_done.record(main)
        e = rr.engine
        split = e.last["grav_split_row"]
        late = ("grav",)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_sph)
            for k in out_names:
                if k not in late and e.out[k].shape == pinned_out[k].shape:
                    pinned_out[k].copy_(e.out[k], non_blocking=True)
            if "density" in pinned_out and \
                    e.fields()["density"].shape == pinned_out["density"].shape:
                pinned_out["density"].copy_(e.fields()["density"], non_blocking=True)
            s_out.wait_event(ev_gh)   # gravity rows [0, split) are final
            for k in late:
                if split > 0 and e.out[k].shape == pinned_out[k].shape:
                    pinned_out[k][:split].copy_(e.out[k][:split], non_blocking=True)
            s_out.wait_event(ev_done)
            for k in late:
                if e.out[k].shape == pinned_out[k].shape:
                    pinned_out[k][split:].copy_(e.out[k][split:], non_blocking=True)
        main.wait_stream(s_out)
        main.synchronize()
        e.check_status(status)

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms_e2e, float(h2d), float(d2h)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t[0].item())
        tt = torch.tensor([float(h2d), float(d2h)], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        h2d, d2h = float(tt[0].item()), float(tt[1].item())
    e2e_value = n_total / (ms_e2e * 1e-3)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    # ---- roofline of the dominant kernel (k_gravity, event-timed live above)
    if n_total > 40_000_000:
        # exact counting pass too large to run untimed next to the rank data:
        # per-particle in-support counts measured at c2 (same sigma/d statistics)
        # (gravity: neighbours within r_cut = 5 d at 2 particles per d^3; a
        # single-species set has half the number density)
        per = {"gravity": 1047.0503, "sph": 81.0037}
        n_gas = meta["n_gas"]
        sph = int(per["sph"] * n_gas)
        g_per = per["gravity"] * (1.0 if species_c == "both" else 0.5)
        counts = {"gravity": int(g_per * n_total), "density": sph, "ncount": sph,
                  "crk": sph, "hydro": max(sph - n_gas, 0),
                  "estimated": "per-particle counts measured exactly at c2 (2x128^3), "
                               "halved for gravity in single-species sets"}
    else:
        counts = pair_counts(p, cfg)
    peak, peak_src = peaks()
    alg_flops = counts["gravity"] * OPCOST["gravity"]
    t_grav = ph.get("k_gravity_max_over_ranks", ph["k_gravity"]) * 1e-3
    achieved = alg_flops / t_grav / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get("gravity_dram_bytes_per_launch")
    roof = {"bound": "fp32", "kernel": "k_gravity (single launch, CUDA events on its stream)",
            "achieved": achieved, "peak": peak * world, "unit": "TFLOP/s",
            "frac": achieved / (peak * world), "traffic": traffic, "peak_source": peak_src,
            "algorithmic_flops_per_launch": alg_flops, "in_support_pairs": counts["gravity"],
            "flops_per_pair": OPCOST["gravity"]}
    step_flops = sum(counts[k] * OPCOST[k] for k in OPCOST)
    roof["step_algorithmic_tflops"] = step_flops / (ms_step * 1e-3) / 1e12
    roof["step_frac"] = roof["step_algorithmic_tflops"] / (peak * world)
    roof["kflop_per_update"] = step_flops / n_total / 1e3
    base = None
    if world == 1 and not args.no_cpu_baseline:
        # one sample of ~10-30 s of host work: 2x the reference arm's per-step
        # fraction (that arm repeats its sample K + W times)
        base = cpu_baseline(p, cfg, frac=min(1.0, 2 * args.cpu_frac),
                            gravity_only=passes != PASS_ALL)
    meta = dict(meta)
    if world > 1:
        meta["parallelism"] = f"spatial cuboids {rr.grid}, overload width {rr.w:.4g}, NCCL all-to-all shell exchange per step"
        # N = 1 runs configs[1] (c2); for the strong-scaling ratio of THIS
        # config, its own 1-GPU line (measured separately) is referenced here
        ref1 = os.path.join(ROOT, "profiles", f"bench_r01_{args.config}_n1.json")
        if os.path.exists(ref1):
            try:
                v1 = json.loads(open(ref1).read().strip().splitlines()[-1])["value"]
                meta["same_config_n1"] = {
                    "value": v1, "source": os.path.relpath(ref1, ROOT),
                    "note": "the N=1 default bench line is c2; same-config strong-scaling "
                            "efficiency = value / (n_gpus * this value)"}
            except Exception:
                pass
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": ("synthetic (Zel'dovich-displaced two-species lattice)" if passes == PASS_ALL
                     else "synthetic (Zel'dovich-displaced dark-matter lattice)"),
            "config": meta, "phases_ms": ph,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": ms_e2e},
            "gpu_launches": int(launches), "roofline": roof, "clocks": clocks.summary(),
            "pair_counts": counts}
    if base is not None:
        line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["cpu_baseline"]["seconds"] = base["seconds"]
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="workload (default: c2 at 1 GPU, c4 at more)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-frac", type=float, default=1 / 16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.config is None:
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        args.config = DEFAULT_CONFIG.get(world, DEFAULT_CONFIG_MULTI)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
