"""Generate the golden vectors that pin the oracle and the CUDA path.

Runs the REFERENCE implementation (hydrobox, /root/reference/pkg/src) in this
container and stores its inputs and outputs as small compressed .npz files in
tests/golden/.  The reference cannot travel to the GPU box; these fixtures do.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every fixture stores raw arrays only (no pickled objects).  Sources for each
recipe are cited inline (hb/ = /root/reference/pkg/src/hydrobox/).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from hydrobox.box import BoxGeometry  # noqa: E402
from hydrobox.checks import _mixed_set  # noqa: E402  (hb/checks.py:90-97)
from hydrobox.cmtree import (InteractionList, assemble_interaction_lists,  # noqa: E402
                             build_mesh_and_leaves)
from hydrobox.config import SimConfig  # noqa: E402
from hydrobox.domain import build_overload, decompose  # noqa: E402
from hydrobox.gravity import (ForceSplit, _optimal_influence, deposit_cic,  # noqa: E402
                              interpolate_force, long_range_potential_energy,
                              short_range_gravity_kernel, solve_long_range)
from hydrobox.hydro import (adapt_smoothing_length, compute_crk_coefficients,  # noqa: E402
                            compute_density, compute_hydro_accel,
                            corrected_interpolate, refresh_eos_columns)
from hydrobox.ic import make_clustered_ic, make_lattice_ic  # noqa: E402
from hydrobox.kernels import (counting_kernel, crk_interp_kernel,  # noqa: E402
                              crk_moments_kernel, density_kernel,
                              gravity_potential_kernel, hydro_force_kernel,
                              neighbor_count_kernel)
from hydrobox.lane import EvalMode, eval_interaction_list, reference_pair_sum  # noqa: E402
from hydrobox.hydro import assign_timestep_levels  # noqa: E402
from hydrobox.insitu import (dbscan_find, encode_halo_catalog, fof_find,  # noqa: E402
                             power_spectrum)
from hydrobox.tiered_io import encode_rank_checkpoint  # noqa: E402
from hydrobox.stepper import ShortRangeContext, subcycle_pm_step, unordered_due_pairs  # noqa: E402

REL, DET = EvalMode.RELAXED, EvalMode.DETERMINISTIC


def particle_arrays(p, prefix=""):
    return {prefix + "pos": p.pos.copy(), prefix + "vel": p.vel.copy(),
            prefix + "mass": p.mass.copy(), prefix + "smoothing": p.smoothing.copy(),
            prefix + "internal_energy": p.internal_energy.copy(),
            prefix + "density": p.density.copy(), prefix + "species": p.species.copy(),
            prefix + "ghost": p.ghost.copy(), prefix + "image_shift": p.image_shift.copy(),
            prefix + "global_id": p.global_id.copy(), prefix + "ghost_src": p.ghost_src.copy(),
            prefix + "timestep_level": p.timestep_level.copy()}


def mesh_arrays(mesh, prefix="mesh_"):
    return {prefix + "leaf_start": mesh.leaf_start, prefix + "leaf_end": mesh.leaf_end,
            prefix + "leaf_lo": mesh.leaf_lo, prefix + "leaf_hi": mesh.leaf_hi,
            prefix + "leaf_ghost_only": mesh.leaf_ghost_only,
            prefix + "leaf_bin": mesh.leaf_bin, prefix + "leaf_level": mesh.leaf_level,
            prefix + "bin_count": mesh.bin_count, prefix + "bin_width": mesh.bin_width,
            prefix + "periodic": mesh.periodic_axis, prefix + "bin_ptr": mesh._bin_ptr,
            prefix + "bin_ids": mesh._bin_ids}


def lane_fixture():
    """check_lane_oracle recipe (hb/checks.py:103-134) for three configs, both modes."""
    box = BoxGeometry(1.0)
    out = {}
    rng = np.random.default_rng(101)
    cfg_ns = []
    for c in range(20):
        n = int(rng.integers(100, 2200))
        cfg_ns.append(n)
    picks = [c for c in range(20) if cfg_ns[c] <= 1300][:3]
    out["configs"] = np.array(picks)
    for c in picks:
        n = cfg_ns[c]
        p = _mixed_set(n, 101 + c, box)
        spacing = 1.0 / n ** (1 / 3)
        reach = min(4.0 * spacing, 0.45)
        mesh = build_mesh_and_leaves(p, box, max(reach, 0.2), 48)
        state = p.state_matrix(5.0 / 3.0)
        ilist = assemble_interaction_lists(mesh, reach, 0)
        k = f"c{c}_"
        out[k + "state"] = state
        out[k + "reach"] = np.float64(reach)
        out[k + "spacing"] = np.float64(spacing)
        out[k + "la"], out[k + "lb"], out[k + "ls"] = ilist.leaf_a, ilist.leaf_b, ilist.shift
        out.update(mesh_arrays(mesh, k + "mesh_"))
        aux = np.zeros((n, 5))
        arng = np.random.default_rng(7 + c)
        aux[:, 0] = arng.normal(size=n)
        aux[:, 1] = arng.uniform(0.5, 1.5, n)
        aux[:, 2:5] = arng.normal(0, 0.3, (n, 3))
        out[k + "aux"] = aux
        kernels = {
            "counting": counting_kernel(reach),
            "gravity": short_range_gravity_kernel(ForceSplit(r_s=reach / 5.0, r_cut=reach),
                                                  spacing / 50),
            "grav_pot": gravity_potential_kernel(reach / 5.0, reach, spacing / 50),
            "density": density_kernel(reach),
            "neighbor_count": neighbor_count_kernel(reach),
            "crk_moments": crk_moments_kernel(reach),
            "hydro": hydro_force_kernel(reach),
            "crk_interp": crk_interp_kernel(reach),
        }
        for name, ker in kernels.items():
            kx = aux if ker.n_aux else None
            for mode, tag in ((REL, "rel"), (DET, "det")):
                res = eval_interaction_list(ker, ilist, state, mesh, mode=mode,
                                            workers=1, aux=kx)
                out[k + f"{name}_{tag}"] = res.values
                if tag == "det":
                    out[k + f"{name}_detint"] = res.int_acc
                out[k + f"{name}_{tag}_counters"] = np.array(
                    [res.counters[x] for x in ("f_evals", "g_evals", "rotations",
                                               "pairs_scheduled", "pairs_in_reach")])
            # worker split (relaxed merge order) for one kernel
            if name == "gravity":
                res3 = eval_interaction_list(ker, ilist, state, mesh, mode=REL, workers=3)
                out[k + "gravity_rel_w3"] = res3.values
            ref, absum = reference_pair_sum(ker, state, box.side_length, mode=REL, aux=kx)
            out[k + f"{name}_allpairs"] = ref
            out[k + f"{name}_allpairs_abs"] = absum
        # mirror evaluation over the unordered list (hb/stepper.py:79-100,136)
        pa, pb, psh, plev = unordered_due_pairs(ilist, mesh)
        out[k + "ua"], out[k + "ub"], out[k + "us"] = pa, pb, psh
        sub = InteractionList(pa, pb, ilist.reach, 0, psh)
        for name in ("gravity", "hydro"):
            ker = kernels[name]
            for mode, tag in ((REL, "rel"), (DET, "det")):
                res = eval_interaction_list(ker, sub, state, mesh, mode=mode, mirror=True)
                out[k + f"{name}_mirror_{tag}"] = res.values
    return out


def mesh_fixture():
    """build_mesh_and_leaves + assemble_interaction_lists (hb/cmtree.py:125-196, 303-337)."""
    box = BoxGeometry(1.0)
    out = {}
    cases = []
    # (a) random mixed set on the bare periodic mesh, leaf size 48
    p = _mixed_set(3000, 77, box)
    cases.append(("rand", p, 0.2, 48, None, None, [0.07, 0.2]))
    # (b) unjittered two-species lattice with (1,1,1) overload: exact coordinate ties
    p = make_lattice_ic(6, box, 0.0, seed=1)
    w = 0.3
    doms = decompose(box, (1, 1, 1), w)
    rs = build_overload(p, doms, box, (1, 1, 1))[0][0]
    cases.append(("lat", rs, 0.32, 64, doms[0].lo - w, doms[0].hi + w, [0.3]))
    # (c) clustered set: deep k-d recursion inside dense bins
    p = make_clustered_ic(10, box, seed=5)
    cases.append(("clu", p, 0.2, 32, None, None, [0.1]))
    # (d) 2x2x1 rank grid: one rank's overloaded working set (non-periodic x,y; periodic z)
    p = make_lattice_ic(8, box, 0.02, seed=3)
    w = 0.15
    doms = decompose(box, (2, 2, 1), w)
    rs = build_overload(p, doms, box, (2, 2, 1))[0][1]
    d1 = doms[1]
    cases.append(("r221", rs, 0.16, 40, d1.lo - w, d1.hi + w, [0.15]))
    for tag, ps, bw, leaf, lo, hi, reaches in cases:
        k = tag + "_"
        out.update(particle_arrays(ps, k + "in_"))
        out[k + "bin_width"] = np.float64(bw)
        out[k + "max_leaf"] = np.int64(leaf)
        out[k + "bounds_lo"] = np.zeros(3) if lo is None else np.asarray(lo, float)
        out[k + "bounds_hi"] = np.ones(3) if hi is None else np.asarray(hi, float)
        q = ps.copy()
        mesh = build_mesh_and_leaves(q, box, bw, leaf, lo, hi)
        out[k + "out_global_id"] = q.global_id.copy()
        out[k + "out_image_shift"] = q.image_shift.copy()
        out[k + "out_ghost_src"] = q.ghost_src.copy()
        out.update(mesh_arrays(mesh, k + "mesh_"))
        # levels for an active-depth list: deterministic pseudo-levels
        lev = (np.arange(mesh.n_leaves) * 7919) % 3
        out[k + "levels"] = lev
        for ri, reach in enumerate(reaches):
            il = assemble_interaction_lists(mesh, reach, 0)
            out[k + f"list{ri}_reach"] = np.float64(reach)
            out[k + f"list{ri}_a"], out[k + f"list{ri}_b"], out[k + f"list{ri}_s"] = \
                il.leaf_a, il.leaf_b, il.shift
        mesh.leaf_level[:] = lev
        il = assemble_interaction_lists(mesh, reaches[0], 1)
        out[k + "listd1_a"], out[k + "listd1_b"], out[k + "listd1_s"] = \
            il.leaf_a, il.leaf_b, il.shift
    return out


def step_fixture():
    """One s=0 force evaluation on a jittered 2x8^3 lattice, (1,1,1) overload
    (SURVEY.md Appendix B recipe; correct ordered paths per SURVEY.md 8c)."""
    box = BoxGeometry(1.0)
    npd = 8
    cfg = SimConfig()
    cfg.n_per_dim = npd
    cfg.pm_grid_n = 4 * npd     # r_cut = 2.5 spacings keeps the 2x8^3 overload legal
    p = make_lattice_ic(npd, box, 0.1 / npd, seed=1234)
    rng = np.random.default_rng(99)
    p.vel = rng.normal(0, 0.05, p.pos.shape)     # exercise the viscosity branch
    p.internal_energy[p.species == 1] = rng.uniform(0.5e-4, 2e-4, int((p.species == 1).sum()))
    split = ForceSplit(r_s=cfg.split_scale, r_cut=cfg.r_cut)
    eps = cfg.softening_for(p.n)
    reach = max(split.r_cut, 2 * p.smoothing.max())
    w = 1.25 * reach
    doms = decompose(box, (1, 1, 1), w)
    rs = build_overload(p, doms, box, (1, 1, 1))[0][0]
    out = {}
    out.update(particle_arrays(rs, "in_"))
    bw = max(cfg.cm_bin_width, reach * (1 + 1e-9))
    lo, hi = doms[0].lo - w, doms[0].hi + w
    out["bin_width"], out["bounds_lo"], out["bounds_hi"] = np.float64(bw), lo, hi
    out["reach"], out["r_s"], out["r_cut"], out["eps"] = (np.float64(reach), np.float64(split.r_s),
                                                          np.float64(split.r_cut), np.float64(eps))
    mesh = build_mesh_and_leaves(rs, box, bw, 256, lo, hi)
    out.update(particle_arrays(rs, "built_"))
    out.update(mesh_arrays(mesh))
    il = assemble_interaction_lists(mesh, reach, 0)
    out["la"], out["lb"], out["ls"] = il.leaf_a, il.leaf_b, il.shift
    st = rs.state_matrix(5 / 3)
    h_max = rs.smoothing.max()
    nc = eval_interaction_list(neighbor_count_kernel(2 * h_max), il, st, mesh, mode=DET,
                               pshift=rs.image_shift)
    out["ncount"] = nc.values[:, 0]
    rho = compute_density(rs, mesh, st, il, mode=REL)
    out["rho_raw"] = rho
    out["density"] = rs.density.copy()
    refresh_eos_columns(st, rs, 5 / 3)
    out["state_eos"] = st.copy()
    crk = compute_crk_coefficients(rs, mesh, st, il, mode=REL)
    out["crk_A"], out["crk_B"], out["crk_fallback"] = crk.A, crk.B, crk.fallback
    out["crk_m0"], out["crk_m1"], out["crk_m2"] = crk.m0, crk.m1, crk.m2
    g = eval_interaction_list(short_range_gravity_kernel(split, eps), il, st, mesh,
                              mode=REL, pshift=rs.image_shift)
    out["grav"] = g.values
    out["grav_counters"] = np.array([g.counters["pairs_scheduled"], g.counters["pairs_in_reach"]])
    f, e, hres = compute_hydro_accel(rs, mesh, st, il, mode=REL, mirror=False)
    out["hydro_force"], out["hydro_edot"] = f, e
    # corrected interpolation of a linear field (hb/hydro.py:162-178)
    fld = 0.3 + rs.pos @ np.array([1.0, -2.0, 0.5])
    out["interp_field"] = fld
    out["interp"] = corrected_interpolate(rs, mesh, st, il, crk, fld, mode=REL)
    return out


def adapt_fixture():
    """adapt_smoothing_length on a jittered gas lattice (hb/hydro.py:199-248)."""
    box = BoxGeometry(1.0)
    p = make_lattice_ic(8, box, 0.15 / 8, seed=21)
    w = 0.3
    doms = decompose(box, (1, 1, 1), w)
    rs = build_overload(p, doms, box, (1, 1, 1))[0][0]
    out = {}
    bw = 0.32
    mesh = build_mesh_and_leaves(rs, box, bw, 64, doms[0].lo - w, doms[0].hi + w)
    out.update(particle_arrays(rs, "in_"))
    out.update(mesh_arrays(mesh))
    out["bin_width"] = np.float64(bw)
    h = adapt_smoothing_length(rs, mesh, lambda: rs.state_matrix(5 / 3), 40, bw, mode=DET)
    out["h_out"] = h.copy()
    return out


def adapt_periodic_fixture():
    """adapt_smoothing_length on a jittered two-species lattice in a bare
    periodic box (no overload shell, so no alias ghosts): the case the
    device-resident iteration serves."""
    box = BoxGeometry(1.0)
    p = make_lattice_ic(12, box, 0.2 / 12, seed=22)
    bw = 0.25
    mesh = build_mesh_and_leaves(p, box, bw, 64)
    out = {}
    out.update(particle_arrays(p, "in_"))
    out.update(mesh_arrays(mesh))
    out["bin_width"] = np.float64(bw)
    h = adapt_smoothing_length(p, mesh, lambda: p.state_matrix(5 / 3), 40, bw, mode=DET)
    out["h_out"] = h.copy()
    return out


def subcycle_fixture():
    """One PM interval of the hierarchical subcycle (hb/stepper.py:103-192) on a
    bare periodic 2x8^3 box (no overload shell, so no same-rank alias ghosts:
    SURVEY.md finding 3 cannot trigger), levels from assign_timestep_levels
    (hb/hydro.py:277-317) with synthetic DM accelerations; run in deterministic
    and relaxed mode from identical inputs."""
    box = BoxGeometry(1.0)
    npd = 8
    p = make_lattice_ic(npd, box, 0.1 / npd, seed=77)
    rng = np.random.default_rng(5)
    p.vel = rng.normal(0, 0.05, p.pos.shape)
    gas = p.species == 1
    p.internal_energy[gas] = rng.uniform(0.5e-2, 2e-2, int(gas.sum()))
    p.accel = rng.normal(0, 1, p.pos.shape) * np.exp(rng.uniform(-2, 3, p.n))[:, None]
    split = ForceSplit(r_s=0.03, r_cut=0.15)
    eps = 1.0 / p.n ** (1 / 3) / 50
    reach = max(split.r_cut, 2 * p.smoothing.max())
    bw = reach * (1 + 1e-9)
    mesh = build_mesh_and_leaves(p, box, bw, 16)
    out = {}
    # dt_pm such that the deepest leaf sits at level 2 (n_fine = 4, 5 boundaries)
    probe = p.copy()
    dt_pm = 1e-3
    for _ in range(60):
        h = assign_timestep_levels(probe, mesh, dt_pm, 0.25, 4, eps, 5 / 3)
        if h.max_level >= 2:
            break
        dt_pm *= 1.5
    hier = assign_timestep_levels(p, mesh, dt_pm, 0.25, 4, eps, 5 / 3)
    out.update(particle_arrays(p, "in_"))
    out["in_accel"] = p.accel.copy()
    out.update(mesh_arrays(mesh))
    out["dt_pm"], out["max_level"], out["n_levels"] = (np.float64(dt_pm), np.int64(hier.max_level),
                                                       np.int64(hier.n_levels))
    out["reach"], out["r_s"], out["r_cut"], out["eps"] = (np.float64(reach), np.float64(split.r_s),
                                                          np.float64(split.r_cut), np.float64(eps))
    for tag, mode in (("det", DET), ("rel", REL)):
        q = p.copy()
        m = build_mesh_and_leaves(q, box, bw, 16)
        m.leaf_level[:] = mesh.leaf_level
        ctx = ShortRangeContext(particles=q, mesh=m, box=box, eos_gamma=5 / 3, reach=reach,
                                mode=mode, gravity_kernel=short_range_gravity_kernel(split, eps),
                                hydro_enabled=True)
        audit = subcycle_pm_step(ctx, hier)
        for k in ("pos", "vel", "internal_energy", "density", "accel"):
            out[f"{tag}_{k}"] = getattr(q, k).copy()
        out[f"{tag}_leaf_lo"], out[f"{tag}_leaf_hi"] = m.leaf_lo.copy(), m.leaf_hi.copy()
        out[f"{tag}_max_quanta"] = np.int64(audit.max_momentum_quanta)
        log = [(r.s, r.depth, lv, n) for r in audit.boundary_log
               for lv, n in sorted(r.pairs_per_level.items())]
        out[f"{tag}_pairs_log"] = np.array(log, dtype=np.int64).reshape(-1, 4)
    return out


def pm_fixture(L=1.0):
    """Long-range PM pipeline (hb/gravity.py:58-245): CIC deposit, alias-optimal
    and naive influence, filtered spectral solve with potential, CIC gather and
    the long-range potential energy, on a jittered 2x8^3 lattice, 16^3 grid,
    in a box of side L."""
    box = BoxGeometry(L)
    p = make_lattice_ic(8, box, 0.2 / 8, seed=404)
    rng = np.random.default_rng(3)
    p.mass = p.mass * rng.uniform(0.5, 1.5, p.n)  # unequal masses exercise the weights
    n = 16
    split = ForceSplit.for_grid(box, n)
    out = {"pos": p.pos.copy(), "mass": p.mass.copy(), "grid_n": np.int64(n), "L": np.float64(L),
           "r_s": np.float64(split.r_s), "r_cut": np.float64(split.r_cut)}
    rho = deposit_cic(p, n, box)
    out["rho"] = rho.values.copy()
    out["d_opt"] = _optimal_influence(n, box, split.r_s).copy()
    for tag in ("optimal", "naive"):
        fields, pot = solve_long_range(rho, split, box, want_potential=True, influence=tag)
        out[f"{tag}_fields"] = np.stack([f.values for f in fields])
        out[f"{tag}_pot"] = pot.values.copy()
        out[f"{tag}_acc"] = interpolate_force(fields, p)
        out[f"{tag}_energy"] = np.float64(long_range_potential_energy(pot, p))
    return out


def _groups_arrays(groups, tag):
    ids = [g.member_ids for g in groups]
    return {f"{tag}_halo_id": np.array([g.halo_id for g in groups], dtype=np.int64),
            f"{tag}_count": np.array([g.count for g in groups], dtype=np.int64),
            f"{tag}_mass": np.array([g.total_mass for g in groups]),
            f"{tag}_center": np.array([g.center for g in groups]).reshape(-1, 3),
            f"{tag}_radius": np.array([g.radius for g in groups]),
            f"{tag}_members": np.concatenate(ids) if ids else np.zeros(0, dtype=np.int64),
            f"{tag}_offsets": np.cumsum([0] + [len(i) for i in ids]).astype(np.int64)}


def fof_fixture():
    """Friends-of-friends and DBSCAN (hb/insitu.py:244-368) on a clustered box,
    single periodic set and (2,2,1) overloaded rank sets (global-id stitching);
    halo catalog bytes (CRC32C footer) and P(k) of its CIC density."""
    box = BoxGeometry(1.0)
    p = make_clustered_ic(16, box, seed=11)
    out = {"pos": p.pos.copy(), "mass": p.mass.copy(), "global_id": p.global_id.copy(),
           "species": p.species.copy()}
    ll = 0.2 / 16
    out["ll"] = np.float64(ll)
    out.update(_groups_arrays(fof_find(p, box, ll, min_members=5), "fof1"))
    w = 2.5 * ll
    doms = decompose(box, (2, 2, 1), w)
    sets = build_overload(p, doms, box, (2, 2, 1))[0]
    for r, rs in enumerate(sets):
        out.update(particle_arrays(rs, f"rank{r}_"))
    out["w"] = np.float64(w)
    out.update(_groups_arrays(fof_find(sets, box, ll, min_members=5, overload_width=w), "fof4"))
    eps = 0.25 / 16
    out["eps"] = np.float64(eps)
    g1, noise1 = dbscan_find(p, box, eps, 6)
    out.update(_groups_arrays(g1, "db1"))
    out["db1_noise"] = noise1
    g4, noise4 = dbscan_find(sets, box, eps, 6, overload_width=w)
    out.update(_groups_arrays(g4, "db4"))
    out["db4_noise"] = noise4
    groups = fof_find(p, box, ll, min_members=5)
    out["catalog"] = np.frombuffer(encode_halo_catalog(groups, 7), dtype=np.uint8).copy()
    rho = deposit_cic(p, 32, box)
    k, pk, cnt = power_spectrum(rho.values, box)
    out["pk_rho"], out["pk_k"], out["pk"], out["pk_counts"] = rho.values, k, pk, cnt
    return out


def ckpt_fixture():
    """HCKP rank checkpoint blob (hb/tiered_io.py:80-96) of one overloaded rank
    set of a 2x8^3 box (ghosts, image shifts, alias sources, timestep levels)."""
    box = BoxGeometry(1.0)
    p = make_lattice_ic(8, box, 0.1 / 8, seed=9)
    rng = np.random.default_rng(4)
    p.vel = rng.normal(0, 0.05, p.pos.shape)
    p.accel = rng.normal(0, 1, p.pos.shape)
    p.timestep_level[:] = rng.integers(0, 4, p.n)
    w = 0.2
    doms = decompose(box, (1, 1, 1), w)
    rs = build_overload(p, doms, box, (1, 1, 1))[0][0]
    out = particle_arrays(rs, "in_")
    out["in_accel"] = rs.accel.copy()
    out["blob"] = np.frombuffer(encode_rank_checkpoint(rs, 12, 3), dtype=np.uint8).copy()
    return out


def levels_fixture():
    """assign_timestep_levels (hb/hydro.py:277-317) on one overloaded rank set
    of a jittered 2x12^3 lattice (ghost-only leaves present): velocities and
    accelerations spread over decades so the gas CFL and DM acceleration
    branches both reach levels 0..3; flat and non-flat; plus the inputs of a
    stiff case (the reference raises StiffStateError)."""
    from hydrobox.errors import StiffStateError
    box = BoxGeometry(1.0)
    p = make_lattice_ic(12, box, 0.2 / 12, seed=21)
    rng = np.random.default_rng(22)
    p.vel = rng.normal(0, 1, p.pos.shape) * 10.0 ** rng.uniform(-3, 0, (p.n, 1))
    p.accel = rng.normal(0, 1, p.pos.shape) * 10.0 ** rng.uniform(-2, 3, (p.n, 1))
    p.internal_energy[p.species == 1] *= 10.0 ** rng.uniform(-1, 1, int((p.species == 1).sum()))
    p.accel[5] = 0.0        # |a| = 0: the 1e-300 floor (dt huge, level 0)
    w = 0.15
    rs = build_overload(p, decompose(box, (2, 1, 1), w), box, (2, 1, 1))[0][0]
    mesh = build_mesh_and_leaves(rs, box, 0.25, 64, bounds_lo=np.array([-w, 0, 0]),
                                 bounds_hi=np.array([0.5 + w, 1, 1]))
    out = particle_arrays(rs, "in_")
    out["in_accel"] = rs.accel.copy()
    out.update(mesh_arrays(mesh))
    eps = 1.0 / 24 / 50
    probe = rs.copy()       # dt_pm such that the deepest level is 3
    assign_timestep_levels(probe, mesh, 1.0, 0.25, 64, eps, 5 / 3)
    dt_pm = 0.9 * 2.0 ** (3 - int(probe.timestep_level.max()))
    out["dt_pm"], out["cfl"], out["eps"] = dt_pm, 0.25, eps
    for tag, flat in (("", False), ("flat_", True)):
        q = rs.copy()
        mesh.leaf_level[:] = 0
        hier = assign_timestep_levels(q, mesh, dt_pm, 0.25, 4, eps, 5 / 3, flat=flat)
        out[tag + "level"] = q.timestep_level.copy()
        out[tag + "leaf_level"] = mesh.leaf_level.copy()
        out[tag + "max_level"] = hier.max_level
    try:
        assign_timestep_levels(rs.copy(), mesh, dt_pm * 64, 0.25, 4, eps, 5 / 3)
        out["stiff_raises"] = 0
    except StiffStateError:
        out["stiff_raises"] = 1
    return out


def main():
    os.makedirs(HERE, exist_ok=True)
    only = set(sys.argv[1:])
    for name, fn in (("lane", lane_fixture), ("mesh", mesh_fixture),
                     ("step", step_fixture), ("adapt", adapt_fixture),
                     ("adapt_periodic", adapt_periodic_fixture),
                     ("subcycle", subcycle_fixture), ("pm", pm_fixture),
                     ("pm_L2", lambda: pm_fixture(2.0)),
                     ("fof", fof_fixture), ("ckpt", ckpt_fixture),
                     ("levels", levels_fixture)):
        if only and name not in only:
            continue
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{path}: {os.path.getsize(path) / 1e3:.0f} kB, {len(data)} arrays")


if __name__ == "__main__":
    sys.exit(main())
