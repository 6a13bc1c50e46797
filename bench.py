#!/usr/bin/env python
"""Benchmark: particle-updates/s of the short-range gravity + CRK-SPH force
evaluation (BASELINE.json metric), on synthetic Zel'dovich-displaced
two-species lattices.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cX] [--impl ours|reference]

Default workload at every N: c4 (2x512^3, configs[3]) -- the largest config that
fits one B200 (158 of 183 GB), the config BASELINE.json names for 2/4/8 GPUs
and for its strong-scaling target, so the driver's 1 -> N ratio divides like
by like.  c2 / c3 (2x128^3 / 2x256^3) and c5 (gravity-only 1024^3 DM, >= 4
GPUs) run with --config.

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
    # stress variant of configs[2]: the reference's own clumped
    # generator (hb/ic.py:137-169, 70% of the particles in 8 Gaussian clumps of
    # sigma L/40), sigma_psi unused; GPU arm only (the CPU reference needs hours)
    "c3k": (128, None, "both", "2x128^3 particles, clustered (hb/ic.py make_clustered_ic): "
                               "neighbour-count imbalance stress case, single B200"),
}
DEVICE_IC_ABOVE = 1 << 29   # particles: displacement field built on the GPU (numpy: ~60 GB/rank)
# default workload at every GPU count (see the module docstring)
DEFAULT_CONFIG = "c4"
SUBBOX_ABOVE = 40_000_000
ZELDOVICH_SEED_CLUSTERED = 3   # CPU samples above this size use an interior sub-box


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
                  region=None, npd: int | None = None):
    """Synthetic workload; local=True (world > 1) materialises only the rows
    rank `rank` owns (identical to selecting them from the full set), so the
    host never holds world copies of a 2x512^3 set; region = (lo, hi) keeps
    only the particles inside that cube (the reference arm's sub-box sample).
    Above DEVICE_IC_ABOVE particles the displacement field is built on the
    GPU (ic.make_zeldovich_ic_device) and a selection is required.  npd: a
    periodic replica of the config on an npd^3 lattice (every scale -- r_s,
    r_cut, h, softening, sigma_psi, bin width -- is relative to the lattice
    spacing, so the per-particle work is the config's; the CPU arms' sample)."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.distributed import rank_grid_for
    from paper_2510_03557_b200.domain import owner_ranks, owner_ranks_torch
    from paper_2510_03557_b200.ic import make_zeldovich_ic, make_zeldovich_ic_device
    from paper_2510_03557_b200.resident import StepConfig
    npd_cfg, sigma, species, desc = CONFIGS[cfg_name]
    npd = npd or npd_cfg
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
    if sigma is None:   # the reference's clustered generator
        from paper_2510_03557_b200.ic import make_clustered_ic
        if select is not None:
            raise ValueError(f"{cfg_name}: the clustered generator is built whole")
        p = make_clustered_ic(npd, box, seed=ZELDOVICH_SEED_CLUSTERED)
    elif on_device:
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
            "smoothing": ("h = 1.3 d as generated (~81 SPH neighbours), not adapted to the 64 of "
                          "SURVEY.md 8d; identical in every arm" if species == "both"
                          else "none (gravity only)"),
            "passes": "all" if species == "both" else "gravity",
            "ic_fft": "cuFFT (GPU)" if on_device else "numpy",
            "r_s": "d", "r_cut": "5 d", "softening": "L/N^(1/3)/50", "max_leaf_size": 256,
            "mesh": "bare periodic box, bin width max(4 PM cells, reach)",
            "bins_per_axis": int(np.floor(1.0 / bin_width)),
            "ic": ("Zel'dovich, seed 2510035570, P(k)~k^-2 exp(-(kd)^2)" if sigma is not None
                   else f"make_clustered_ic(seed={ZELDOVICH_SEED_CLUSTERED})"),
            "l2": "working set > 126 MB L2 (no flush needed)"}
    return p, cfg, meta


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_step(p, cfg, bounds=None, gravity_only: bool = False,
                       threads: int | None = None) -> dict:
    """One COMPLETE force evaluation of set p by the reference algorithm on the
    host cores: the oracle/ C restatement, pinned bitwise to the reference
    (tests/test_oracle_golden.py), with the reference driver's schedule --
    build_mesh_and_leaves, assemble_interaction_lists, one neighbour-count
    pass, compute_density, refresh_eos_columns, compute_crk_coefficients
    (moments + 3x3 solve), then gravity and hydro over the unordered due pairs
    in mirror mode (hb/stepper.py:113-192).  Nothing is
    sampled or extrapolated: the returned rate is owned rows / wall time.
    bounds: (lo, hi) of a bounded (rank-domain) mesh, else the periodic box."""
    from oracle import oracle as O
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.kernels import (crk_moments_kernel, density_kernel,
                                               hydro_force_kernel, neighbor_count_kernel)
    threads = threads or os.cpu_count() or 1
    O.set_threads(threads)
    L = cfg.box.side_length
    sec = {}
    t_all = time.perf_counter()
    t0 = time.perf_counter()
    blo, bhi = bounds if bounds is not None else (None, None)
    m = O.build_mesh(p.pos, p.image_shift, p.ghost, L, cfg.bin_width, cfg.max_leaf_size,
                     bounds_lo=blo, bounds_hi=bhi)
    sec["build"] = time.perf_counter() - t0
    gas = p.species == 1
    h_max = float(p.smoothing[gas].max()) if np.any(gas) else 0.0
    reach = max(cfg.r_cut, 2 * h_max)
    t0 = time.perf_counter()
    la, lb, ls = O.assemble(m, L, reach)
    sec["list"] = time.perf_counter() - t0
    perm = m["perm"]
    pshift = p.image_shift[perm]
    pshift = pshift if np.any(pshift) else None
    st = O.state_matrix(p.pos[perm], p.vel[perm], p.mass[perm], p.smoothing[perm],
                        p.density[perm], p.internal_energy[perm], p.species[perm], cfg.eos_gamma)
    args = (m["leaf_start"], m["leaf_end"], L)

    def ev(name, ker, A, B, S, mode="relaxed", mirror=False):
        t = time.perf_counter()
        v, _, _, err = O.eval_pairs(ker, A, B, S, st, *args, mode=mode, workers=threads,
                                    mirror=mirror, pshift=pshift)
        sec[name] = time.perf_counter() - t
        if err:
            raise RuntimeError(f"reference step: {name} raised {err}")
        return v

    if not gravity_only:
        ev("ncount", neighbor_count_kernel(2 * h_max), la, lb, ls, mode="deterministic")
        rho = ev("density", density_kernel(2 * h_max), la, lb, ls)
        t = time.perf_counter()
        gp = gas[perm]
        # write-back for gas rows of receiver leaves only (hb/hydro.py:73-80)
        active_row = np.repeat(~np.asarray(m["leaf_ghost_only"], bool),
                               m["leaf_end"] - m["leaf_start"])
        dens = np.where(gp & active_row, rho[:, 0], st[:, 8])
        O.refresh_eos(st, dens, p.internal_energy[perm], cfg.eos_gamma)
        sec["eos"] = time.perf_counter() - t
        mom = ev("crk", crk_moments_kernel(2 * h_max), la, lb, ls)
        t = time.perf_counter()
        O.crk_solve(mom, gp)
        sec["crk_solve"] = time.perf_counter() - t
    t = time.perf_counter()
    ua, ub, us, _ = O.unordered_due_pairs(la, lb, ls, m["leaf_start"].shape[0])
    sec["unordered"] = time.perf_counter() - t
    gk = short_range_gravity_kernel(ForceSplit(r_s=cfg.r_s, r_cut=cfg.r_cut), cfg.softening)
    ev("gravity", gk, ua, ub, us, mirror=True)
    if not gravity_only:
        ev("hydro", hydro_force_kernel(2 * h_max, cfg.visc_alpha, cfg.visc_beta), ua, ub, us,
           mirror=True)
    total = time.perf_counter() - t_all
    sec["total"] = total
    n_owned = int(np.count_nonzero(p.ghost == 0))
    return {"value": n_owned / total, "unit": UNIT, "cores": threads, "kind": "port",
            "n_owned": n_owned, "n_rows": int(p.n), "seconds": sec}


def reference_sample(cfg_name: str, npd_sample: int):
    """The CPU arms' bounded workload: a periodic replica of config cfg_name on
    an npd_sample^3 lattice (make_workload(npd=...): the same generator, every
    scale relative to the lattice spacing, so each particle sees the config's
    neighbourhood -- ~1047 gravity sources within r_cut and ~81 SPH neighbours
    at 2 x npd^3 -- and, like the GPU arm at N = 1, a bare periodic mesh with
    no shell).  Returns (p, cfg, meta of the FULL config + the sample, desc)."""
    npd_cfg, _, species, _ = CONFIGS[cfg_name]
    npd = min(int(npd_sample), npd_cfg)
    p, cfg, meta = make_workload(cfg_name, npd=npd)
    k = 2 if species == "both" else 1
    d = 1.0 / npd_cfg
    meta = dict(meta, n_particles=k * npd_cfg ** 3, n_gas=npd_cfg ** 3 if k == 2 else 0,
                n_per_dim=npd_cfg,
                bins_per_axis=int(np.floor(1.0 / max(2.0 * d, 5.0 * d * (1 + 1e-9)))))
    desc = (f"periodic {'2x' if k == 2 else ''}{npd}^3 replica of the {cfg_name} workload "
            f"({p.n} particles, all owned): the same generator with sigma_psi, h, r_s, r_cut, "
            f"softening and bin width relative to the lattice spacing, so the same "
            f"per-particle work")
    meta["cpu_sample"] = {"n_per_dim": npd, "n_particles": int(p.n), "kind": "periodic replica"}
    return p, cfg, meta, None, desc


# lattice of the CPU samples.  npd = 5 k + 1 keeps the replica's bin width
# (1 / floor(npd / 5) of the box, hb/driver.py:147-150) within 2% of the
# full configs' 5.02 d (the bin width sets the leaf size and so the scheduled
# pairs per particle).  A complete reference step of 2x46^3 takes ~7 s on the
# GPU box's 16 host cores: the driver's K + W = 25 steps run in ~3 minutes.
CPU_SAMPLE_NPD = {"both": 46, "dm": 71}
CPU_BASELINE_NPD = {"both": 51, "dm": 81}   # the GPU arm's single cpu_baseline step


def run_reference_arm(args):
    """--impl reference: the reference algorithm on the host cores, on a
    bounded sample of the same workload (the sub-box above), K timed complete
    steps after W untimed ones.  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    species = CONFIGS[args.config][2]
    if CONFIGS[args.config][1] is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"{args.config}: clump size is a fixed fraction of the box, so no "
                          "bounded replica carries the per-particle work, and the whole set "
                          "needs hours on the host"}), flush=True)
        return 0
    npd = getattr(args, "cpu_npd", None) or CPU_SAMPLE_NPD[species]
    p, cfg, meta, bounds, desc = reference_sample(args.config, npd)
    gonly = species == "dm"
    for _ in range(args.warmup):
        cpu_reference_step(p, cfg, bounds, gravity_only=gonly)
    steps = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        steps.append(cpu_reference_step(p, cfg, bounds, gravity_only=gonly))
    wall = time.perf_counter() - t0
    n_owned = steps[0]["n_owned"]
    ms_step = wall / args.steps * 1e3
    v = n_owned / (ms_step * 1e-3)
    phases = {k: float(np.median([x["seconds"][k] for x in steps])) for k in steps[0]["seconds"]}
    cores = steps[0]["cores"]
    meta = dict(meta)
    meta["updates_per_step"] = n_owned
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": meta,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "cpu_model": cpu_model(), "extrapolated": False,
                             "sample": desc + "; every step a complete force evaluation "
                                              "(no list sampling)",
                             "seconds_per_phase": phases},
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

    # ---- exact pair counts: an untimed accounting pass on every rank (the
    # gravity count re-steps the rank set with HB_PASS_COUNT_ONLY; SPH counts
    # are the step's own exact neighbour counts, r <= 2 h_i gas-gas incl. self)
    eng = rr if world == 1 else rr.engine
    fl = eng.fields()
    own = fl["ghost"] == 0
    sph_in = n_gas_own = 0
    if passes == PASS_ALL:
        gown = own & (fl["species"] == 1)
        sph_in = int(eng.out["ncount"][:eng.n][gown].sum().item())
        n_gas_own = int(gown.sum().item())
    t_cnt = time.perf_counter()
    g_pairs = eng.gravity_pair_count(owned_only=world > 1)
    t_cnt = time.perf_counter() - t_cnt
    if dist:
        t = torch.tensor([g_pairs, sph_in, n_gas_own], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        g_pairs, sph_in, n_gas_own = (int(x) for x in t.tolist())
    counts = {"gravity": g_pairs, "density": sph_in, "ncount": sph_in, "crk": sph_in,
              "hydro": max(sph_in - n_gas_own, 0),
              "how": "exact: gravity = ordered (i, j != i) pairs with r <= r_cut from the "
                     "device counting pass (float64 re-check at the threshold); SPH = the "
                     "step's neighbour counts (r <= 2 h_i, gas-gas, incl. self; hydro "
                     "excludes self; uniform h)",
              "count_pass_s": t_cnt}
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    # ---- roofline of the dominant kernel (k_gravity, event-timed live above)
    peak, peak_src = peaks()
    alg_flops = counts["gravity"] * OPCOST["gravity"]
    t_grav = ph.get("k_gravity_max_over_ranks", ph["k_gravity"]) * 1e-3
    achieved = alg_flops / t_grav / 1e12
    # ncu evidence for this config's k_gravity (profiles/traffic_<config>.json,
    # from one `ncu --set full` capture): DRAM bytes per launch and the executed
    # FP32 operations (fadd + fmul + 2 ffma, the paper's counting rule,
    # PAPER.md:238) -- the latter over the live kernel time gives the executed
    # FP32 rate next to the algorithmic one
    traffic, fp32_ops = None, None
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tf):
        rec = json.load(open(tf))
        traffic = rec.get("gravity_dram_bytes_per_launch")
        fp32_ops = rec.get("gravity_fp32_ops_per_launch")
    roof = {"bound": "fp32", "kernel": "k_gravity (single launch, CUDA events on its stream)",
            "achieved": achieved, "peak": peak * world, "unit": "TFLOP/s",
            "frac": achieved / (peak * world), "traffic": traffic, "peak_source": peak_src,
            "algorithmic_flops_per_launch": alg_flops, "in_support_pairs": counts["gravity"],
            "flops_per_pair": OPCOST["gravity"]}
    if fp32_ops:
        roof["executed_fp32_tflops"] = fp32_ops / t_grav / 1e12
        roof["executed_fp32_frac"] = roof["executed_fp32_tflops"] / (peak * world)
        roof["executed_per_algorithmic"] = fp32_ops / alg_flops
    step_flops = sum(counts[k] * OPCOST[k] for k in OPCOST)
    roof["step_algorithmic_tflops"] = step_flops / (ms_step * 1e-3) / 1e12
    roof["step_frac"] = roof["step_algorithmic_tflops"] / (peak * world)
    roof["kflop_per_update"] = step_flops / n_total / 1e3
    base = None
    if world == 1 and not args.no_cpu_baseline and CONFIGS[args.config][1] is not None:
        # one complete reference step on a bounded replica of this workload
        # (~10 s on the host cores), after the GPU timings
        q, qcfg, _, _, desc = reference_sample(args.config, CPU_BASELINE_NPD[species_c])
        base = cpu_reference_step(q, qcfg, None, gravity_only=passes != PASS_ALL)
        base["sample"] = "one complete force evaluation of a " + desc
        base["cpu_model"] = cpu_model()
        base["extrapolated"] = False
    meta = dict(meta)
    if world > 1:
        meta["parallelism"] = f"spatial cuboids {rr.grid}, overload width {rr.w:.4g}, NCCL all-to-all shell exchange per step"
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
        line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                     "cpu_model", "extrapolated")}
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
                    help="workload (default: c4 at every GPU count)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-npd", type=int, default=None,
                    help="lattice of the CPU reference sample (default: CPU_SAMPLE_NPD)")
    args = ap.parse_args()
    if args.config is None:
        args.config = DEFAULT_CONFIG
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
