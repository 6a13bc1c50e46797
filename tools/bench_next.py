"""Measurements of the §8(f) rows built on top of the force path (1 GPU):

  pm        long-range kick at the c2 workload: 2x128^3 particles on the
            pm_grid_n = 2 npd = 256^3 grid (CIC deposit, cuFFT R2C, spectral
            multiply, 3 C2R, CIC gather), CUDA events, median of --reps
  subcycle  one PM interval of the hierarchical integrator (SubcycleEngine) on
            a 2 x npd^3 Zel'dovich box with leaf levels from
            assign_timestep_levels (dt_pm chosen for a 3-level hierarchy)
  fof       FOF (ll = 0.2 d, >= 10 members) and DBSCAN on a 2 x npd^3
            clustered box (device sweeps + host group statistics)
  ckpt      HCKP encode of the c2 rank state from device fields; device CRC32C
            bandwidth over 512 MiB
  adapt     adapt_smoothing_length to 64 neighbours from h = 1.3 d at c1 and c2
  c5rank    (--only c5rank) configs[4]'s per-rank gravity sweep of the 8-GPU
            decomposition on one GPU

    python tools/bench_next.py [--npd 128] [--sub-npd 64] [--reps 5]
Prints one JSON line per measurement."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def bench_pm(npd, reps):
    import numpy as np
    import torch
    from bench import make_workload
    from paper_2510_03557_b200 import gravity as G
    p, cfg, meta = make_workload("c2" if npd == 128 else "c1")
    box = cfg.box
    n = 2 * npd
    split = G.ForceSplit.for_grid(box, n)
    solver = G.LongRangeSolver(n, split, box)
    pos = torch.from_numpy(np.ascontiguousarray(p.pos)).cuda()
    mass = torch.from_numpy(np.ascontiguousarray(p.mass)).cuda()
    t0 = time.perf_counter()
    G.optimal_influence_device(n, box, split.r_s)
    torch.cuda.synchronize()
    t_infl = time.perf_counter() - t0
    stages = {"deposit": [], "solve": [], "gather": [], "total": []}
    for _ in range(reps + 2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        rho = G.deposit_cic_device(pos, mass, n, box)
        ev[1].record()
        fields, pot = G.solve_long_range_device(rho, split, box, False)
        ev[2].record()
        acc = G.interpolate_device(fields, pos, box.side_length / n)
        ev[3].record()
        torch.cuda.synchronize()
        for k, (a, b) in zip(stages, ((0, 1), (1, 2), (2, 3), (0, 3))):
            stages[k].append(ev[a].elapsed_time(ev[b]))
    med = {k: float(np.median(v[2:])) for k, v in stages.items()}
    mom = float((acc * mass[:, None]).sum(dim=0).abs().max() /
                (acc.abs() * mass[:, None]).sum())
    return {"measurement": "pm_long_range_kick", "n_particles": int(p.n), "grid": n,
            "ms": med, "particles_per_s": p.n / (med["total"] * 1e-3),
            "influence_setup_s": t_infl, "momentum_residual_rel": mom,
            "note": "float64 throughout; FFTs are cuFFT (torch.fft); influence cached per grid"}


def bench_subcycle(npd, reps):
    import numpy as np
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import build_mesh_and_leaves
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.hydro import assign_timestep_levels
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.lane import EvalMode
    from paper_2510_03557_b200.stepper import ShortRangeContext, SubcycleEngine
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(npd, box, 0.05)
    rng = np.random.default_rng(1)
    p.internal_energy[p.species == 1] = 1e-2
    p.accel = rng.normal(0, 1, p.pos.shape) * np.exp(rng.uniform(-2, 3, p.n))[:, None]
    split = ForceSplit.for_grid(box, 2 * npd)
    eps = 1.0 / p.n ** (1 / 3) / 50
    reach = max(split.r_cut, 2 * float(p.smoothing.max()))
    mesh = build_mesh_and_leaves(p, box, reach * (1 + 1e-9), 256)
    dt_pm = 1e-3
    for _ in range(80):
        hier = assign_timestep_levels(p.copy(), mesh, dt_pm, 0.25, 4, eps, 5 / 3)
        if hier.max_level >= 2:
            break
        dt_pm *= 1.5
    hier = assign_timestep_levels(p, mesh, dt_pm, 0.25, 4, eps, 5 / 3)
    out = {}
    for mode in (EvalMode.DETERMINISTIC, EvalMode.RELAXED):
        ctx = ShortRangeContext(particles=p, mesh=mesh, box=box, eos_gamma=5 / 3, reach=reach,
                                mode=mode, gravity_kernel=short_range_gravity_kernel(split, eps))
        times = []
        for _ in range(reps):
            eng = SubcycleEngine(ctx)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            audit = eng.run(hier)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        out[mode] = {"s_per_interval": float(np.median(times)),
                     "boundaries": audit.n_boundaries, "max_momentum_quanta":
                     audit.max_momentum_quanta,
                     "pairs_per_boundary": [sum(r.pairs_per_level.values())
                                            for r in audit.boundary_log]}
    levels = np.bincount(mesh.leaf_level, minlength=hier.max_level + 1).tolist()
    return {"measurement": "subcycle_interval", "n_particles": int(p.n), "n_fine": hier.n_fine,
            "leaf_levels": levels, "modes": out,
            "note": "wall time of SubcycleEngine.run (device-resident), compat pair engine "
                    "(hb_eval_pairs) per level"}


def bench_fof(npd, reps):
    import numpy as np
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_clustered_ic
    from paper_2510_03557_b200.insitu import dbscan_find, fof_find
    box = BoxGeometry(1.0)
    p = make_clustered_ic(npd, box, seed=11)  # Gaussian clumps over a floor (hb/ic.py:137)
    ll = 0.2 / npd
    res = {}
    for name, fn in (("fof", lambda: fof_find(p, box, ll, min_members=10)),
                     ("dbscan", lambda: dbscan_find(p, box, ll, 8))):
        fn()
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        groups = out[0] if isinstance(out, tuple) else out
        res[name] = {"s": float(np.median(ts)), "groups": len(groups)}
    return {"measurement": "insitu_cluster_finding", "n_particles": int(p.n),
            "linking_length": "0.2 d", "results": res,
            "note": "wall time incl. host group statistics and H2D of positions"}


def bench_ckpt(npd, reps):
    import numpy as np
    import torch
    from bench import make_workload
    from paper_2510_03557_b200 import _native as N
    from paper_2510_03557_b200.checkpoint import crc32c_device, encode_rank_checkpoint_device
    p, cfg, meta = make_workload("c2" if npd == 128 else "c1")
    fields = {k: N.dev(np.ascontiguousarray(getattr(p, k))) for k in (
        "pos", "vel", "mass", "smoothing", "internal_energy", "density", "species", "ghost",
        "image_shift", "global_id", "ghost_src", "timestep_level", "accel")}
    big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda").random_(0, 255)
    crc32c_device(big)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        crc32c_device(big)
    ev1.record()
    torch.cuda.synchronize()
    crc_gbs = big.numel() * reps / (ev0.elapsed_time(ev1) * 1e-3) / 1e9
    blob = encode_rank_checkpoint_device(fields, 1, 0)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blob = encode_rank_checkpoint_device(fields, 1, 0)
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    return {"measurement": "hckp_encode", "n_particles": int(p.n), "blob_bytes": len(blob),
            "encode_s": t, "encode_gbs": len(blob) / t / 1e9, "device_crc32c_gbs": crc_gbs,
            "note": "encode = device column conversion + 22 device CRCs + assembly + one "
                    "D2H into pinned memory (PCIe-bound)"}


def bench_adapt(npd, reps):
    """adapt_smoothing_length (hb/hydro.py:199-248; the reference's largest
    CPU cost, 47-48 s at 2x32^3 on 8 threads) to 64 neighbours from h = 1.3 d:
    iterations and wall time, counts on the GPU (deterministic mode)."""
    import numpy as np
    import torch
    from bench import make_workload
    from paper_2510_03557_b200.cmtree import build_mesh_and_leaves
    from paper_2510_03557_b200.hydro import adapt_smoothing_length
    from paper_2510_03557_b200.lane import EvalMode
    out = {}
    for name in ("c1", "c2" if npd == 128 else "c1"):
        p0, cfg, meta = make_workload(name)
        ts, iters = [], None
        for _ in range(max(1, reps)):
            p = p0.copy()
            mesh = build_mesh_and_leaves(p, cfg.box, cfg.bin_width, cfg.max_leaf_size)
            from paper_2510_03557_b200 import lane as LN
            calls = {"n": 0}
            inner = LN.eval_on_device

            def counting(*a, **k):   # one count evaluation per iteration
                calls["n"] += 1
                return inner(*a, **k)
            LN.eval_on_device = counting
            try:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                h = adapt_smoothing_length(p, mesh, lambda: p.state_matrix(cfg.eos_gamma), 64,
                                           cfg.bin_width, mode=EvalMode.DETERMINISTIC)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            finally:
                LN.eval_on_device = inner
            iters = calls["n"]
        gas = p.species == 1
        out[name] = {"n_particles": int(p.n), "s": float(np.median(ts)), "iterations": iters,
                     "h_over_d_median": float(np.median(h[gas]) * meta["n_per_dim"])}
        if name == "c2":
            break
    return {"measurement": "adapt_smoothing_length", "target_neighbours": 64, "results": out,
            "note": "state, list and leaf ranges resident on the GPU; per iteration the h "
                    "column is refreshed, counts read back, and h updated in numpy as the "
                    "reference does (bit-identical); reference CPU: 47-48 s at c1, 8 threads"}


def bench_c5_rank(reps):
    """configs[4] (gravity-only 1024^3 DM) per-rank work of its 8-GPU
    decomposition, on one GPU: an interior cube of 1/8 of the volume (134 M
    owned particles, the size of one rank of 2x2x2) plus its r_cut shell as
    ghosts on a bounded mesh, PASS_GRAVITY, ghost-only tiles skipped.  The full
    c5 run needs >= 8 GPUs (about 193 GB per rank at 4)."""
    import numpy as np
    import torch
    from bench import (CONFIGS, OPCOST, make_workload, peaks, subbox_region, subbox_sample)
    from paper_2510_03557_b200.resident import PASS_GRAVITY, ResidentRank, StepConfig
    npd = CONFIGS["c5"][0]
    n_all = npd ** 3
    a, side, reach = subbox_region(1.0, 5.0 / npd, n_all, 0.0, n_target=n_all // 8)
    t0 = time.perf_counter()
    p, cfg, meta = make_workload("c5", region=(a - reach, a + side + reach))
    q, lo, hi = subbox_sample(p, cfg, n_target=n_all // 8, n_all=n_all)
    del p
    t_ic = time.perf_counter() - t0
    n_own = int(np.count_nonzero(q.ghost == 0))
    rcfg = StepConfig(box=cfg.box, bin_width=cfg.bin_width, max_leaf_size=256, r_s=cfg.r_s,
                      r_cut=cfg.r_cut, softening=cfg.softening, bounds_lo=lo, bounds_hi=hi)
    rk = ResidentRank(q, rcfg, gravity_only=True, owned_targets=True)
    for _ in range(2):
        rk.step(PASS_GRAVITY)
    torch.cuda.synchronize()
    ms, kg = [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rk.step(PASS_GRAVITY, timing=True)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        kg.append(rk.last["ms_phase"]["k_gravity"])
    t = float(np.median(ms))
    t_k = float(np.median(kg))
    pairs = 1047.0503 / 2 * n_own          # per-particle in-support count (bench.py)
    peak, _ = peaks()
    return {"measurement": "c5_rank_gravity_sweep", "n_owned": n_own, "n_rows": int(q.n),
            "ms_per_step": t, "updates_per_s_per_gpu": n_own / (t * 1e-3),
            "k_gravity_ms": t_k,
            "k_gravity_fp32_frac": pairs * OPCOST["gravity"] / (t_k * 1e-3) / 1e12 / peak,
            "ic_s": t_ic,
            "note": "one rank's domain of the 2x2x2 decomposition (interior cube, no exchange); "
                    "8 such ranks = the full 1.07 G step minus the shell exchange"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--npd", type=int, default=128)
    ap.add_argument("--sub-npd", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default=None, help="one of pm, subcycle, fof, ckpt, adapt")
    args = ap.parse_args()
    if args.only == "adapt":
        print(json.dumps(bench_adapt(args.npd, max(1, args.reps // 2))))
        return
    if args.only == "fof":
        print(json.dumps(bench_fof(args.npd, max(1, args.reps // 2))))
        return
    if args.only == "c5rank":
        print(json.dumps(bench_c5_rank(args.reps)))
        return
    print(json.dumps(bench_pm(args.npd, args.reps)))
    print(json.dumps(bench_subcycle(args.sub_npd, max(1, args.reps // 2))))
    print(json.dumps(bench_fof(args.npd, max(1, args.reps // 2))))
    print(json.dumps(bench_ckpt(args.npd, args.reps)))
    print(json.dumps(bench_adapt(args.npd, max(1, args.reps // 2))))


if __name__ == "__main__":
    main()
