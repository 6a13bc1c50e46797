"""GPU parity: the CUDA engine against the reference's golden vectors and the
pinned C oracle.  Integer outputs (leaves, permutations, lists, counts,
pairs_in_reach) must be bit-exact; floating outputs meet the FP32 tolerance
stated in tolerances.py (normalised by the reference's own sum_j |phi_ij|)."""
import numpy as np
import pytest

from tests.conftest import MeshView
from tests.test_oracle_golden import KERNELS, make_kernel
from tests.tolerances import assert_fp32_close

pytestmark = pytest.mark.gpu

INTEGER_KERNELS = ("counting", "neighbor_count")


def particle_set(g, prefix):
    from paper_2510_03557_b200.particles import FIELD_SPECS, ParticleSet
    n = g[prefix + "pos"].shape[0]
    p = ParticleSet(n)
    for name, _, _ in FIELD_SPECS:
        if prefix + name in g:
            setattr(p, name, np.array(g[prefix + name]))
    return p


@pytest.mark.parametrize("case", ["rand", "lat", "clu", "r221"])
def test_gpu_mesh_and_lists_bitwise(golden, case):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    g = golden("mesh")
    k = case + "_"
    p = particle_set(g, k + "in_")
    mesh = build_mesh_and_leaves(p, BoxGeometry(1.0), float(g[k + "bin_width"]),
                                 int(g[k + "max_leaf"]), g[k + "bounds_lo"], g[k + "bounds_hi"])
    np.testing.assert_array_equal(p.global_id, g[k + "out_global_id"])
    np.testing.assert_array_equal(p.image_shift, g[k + "out_image_shift"])
    np.testing.assert_array_equal(p.ghost_src, g[k + "out_ghost_src"])
    for f in ("leaf_start", "leaf_end", "leaf_lo", "leaf_hi", "leaf_ghost_only", "leaf_bin"):
        np.testing.assert_array_equal(getattr(mesh, f), g[k + "mesh_" + f], err_msg=f)
    np.testing.assert_array_equal(mesh._bin_ptr, g[k + "mesh_bin_ptr"])
    ri = 0
    while k + f"list{ri}_a" in g:
        il = assemble_interaction_lists(mesh, float(g[k + f"list{ri}_reach"]), 0)
        np.testing.assert_array_equal(il.leaf_a, g[k + f"list{ri}_a"])
        np.testing.assert_array_equal(il.leaf_b, g[k + f"list{ri}_b"])
        np.testing.assert_array_equal(il.shift, g[k + f"list{ri}_s"])
        ri += 1
    mesh.leaf_level[:] = g[k + "levels"]
    il = assemble_interaction_lists(mesh, float(g[k + "list0_reach"]), 1)
    np.testing.assert_array_equal(il.leaf_a, g[k + "listd1_a"])
    np.testing.assert_array_equal(il.leaf_b, g[k + "listd1_b"])
    np.testing.assert_array_equal(il.shift, g[k + "listd1_s"])


@pytest.mark.parametrize("name", KERNELS)
def test_gpu_lane_kernels(golden, oracle, name):
    from paper_2510_03557_b200.cmtree import InteractionList
    from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        st = g[k + "state"]
        ker = make_kernel(name, float(g[k + "reach"]), float(g[k + "spacing"]))
        aux = g[k + "aux"] if ker.n_aux else None
        mesh = MeshView(g, k + "mesh_")
        il = InteractionList(g[k + "la"], g[k + "lb"], ker.reach, 0, g[k + "ls"])
        res = eval_interaction_list(ker, il, st, mesh, mode=EvalMode.RELAXED, aux=aux)
        ref_c = g[k + f"{name}_rel_counters"]
        got_c = [res.counters[x] for x in ("f_evals", "g_evals", "rotations", "pairs_scheduled",
                                           "pairs_in_reach")]
        np.testing.assert_array_equal(got_c, ref_c, err_msg="counters")
        ref = g[k + f"{name}_rel"]
        if name in INTEGER_KERNELS:
            np.testing.assert_array_equal(res.values, ref)
            det = eval_interaction_list(ker, il, st, mesh, mode=EvalMode.DETERMINISTIC, aux=aux)
            np.testing.assert_array_equal(det.values, g[k + f"{name}_det"])
            np.testing.assert_array_equal(det.int_acc, g[k + f"{name}_detint"])
        else:
            absum = oracle.eval_abs_sums(ker, g[k + "la"], g[k + "lb"], g[k + "ls"], st,
                                         mesh.leaf_start, mesh.leaf_end, 1.0, aux=aux)
            assert_fp32_close(res.values, ref, absum, what=f"{name} c{c}")
            # deterministic mode: int64 quanta of the FP32 pair terms
            det = eval_interaction_list(ker, il, st, mesh, mode=EvalMode.DETERMINISTIC, aux=aux)
            assert_fp32_close(det.values, g[k + f"{name}_det"], absum, what=f"{name} det c{c}")


@pytest.mark.parametrize("name", ["gravity", "hydro"])
def test_gpu_mirror_equals_ordered(golden, oracle, name):
    """Mirror evaluation over unordered pairs == reference mirror output."""
    from paper_2510_03557_b200.cmtree import InteractionList
    from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        ker = make_kernel(name, float(g[k + "reach"]), float(g[k + "spacing"]))
        mesh = MeshView(g, k + "mesh_")
        il = InteractionList(g[k + "ua"], g[k + "ub"], ker.reach, 0, g[k + "us"])
        res = eval_interaction_list(ker, il, g[k + "state"], mesh, mode=EvalMode.RELAXED,
                                    mirror=True)
        absum = oracle.eval_abs_sums(ker, g[k + "ua"], g[k + "ub"], g[k + "us"], g[k + "state"],
                                     mesh.leaf_start, mesh.leaf_end, 1.0, mirror=True)
        assert_fp32_close(res.values, g[k + f"{name}_mirror_rel"], absum, what=f"mirror {name}")


def test_gpu_step_fixture(golden, oracle):
    """Overloaded 2x8^3 lattice: density, CRK, gravity, hydro, counts."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.hydro import (compute_crk_coefficients, compute_density,
                                             compute_hydro_accel, corrected_interpolate,
                                             refresh_eos_columns)
    from paper_2510_03557_b200.kernels import hydro_force_kernel, neighbor_count_kernel
    from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
    g = golden("step")
    box = BoxGeometry(1.0)
    p = particle_set(g, "in_")
    mesh = build_mesh_and_leaves(p, box, float(g["bin_width"]), 256, g["bounds_lo"],
                                 g["bounds_hi"])
    np.testing.assert_array_equal(p.global_id, g["built_global_id"])
    il = assemble_interaction_lists(mesh, float(g["reach"]), 0)
    np.testing.assert_array_equal(il.leaf_a, g["la"])
    np.testing.assert_array_equal(il.leaf_b, g["lb"])
    st = p.state_matrix(5 / 3)
    nc = eval_interaction_list(neighbor_count_kernel(2 * p.smoothing.max()), il, st, mesh,
                               mode=EvalMode.DETERMINISTIC, pshift=p.image_shift)
    np.testing.assert_array_equal(nc.values[:, 0], g["ncount"])
    rho = compute_density(p, mesh, st, il, mode=EvalMode.RELAXED)
    rel = np.abs(rho - g["rho_raw"]) / np.maximum(np.abs(g["rho_raw"]), 1e-300)
    gas = p.species == 1
    assert np.median(rel[gas]) <= 1e-6 and np.quantile(rel[gas], 0.999) <= 1e-5, rel[gas].max()
    np.testing.assert_allclose(p.density, g["density"], rtol=1e-5, atol=0)
    refresh_eos_columns(st, p, 5 / 3)
    crk = compute_crk_coefficients(p, mesh, st, il, mode=EvalMode.RELAXED)
    ok = gas & (g["crk_m0"] > 0)
    np.testing.assert_array_equal(crk.fallback, g["crk_fallback"])
    relA = np.abs(crk.A - g["crk_A"])[ok] / np.abs(g["crk_A"][ok])
    assert np.median(relA) <= 1e-6 and np.quantile(relA, 0.999) <= 1e-5, relA.max()
    dB = (np.abs(crk.B - g["crk_B"]).max(axis=1) * p.smoothing)[ok]
    assert dB.max() <= 1e-5, dB.max()
    split = ForceSplit(r_s=float(g["r_s"]), r_cut=float(g["r_cut"]))
    gk = short_range_gravity_kernel(split, float(g["eps"]))
    grav = eval_interaction_list(gk, il, st, mesh, mode=EvalMode.RELAXED, pshift=p.image_shift)
    absg = oracle.eval_abs_sums(gk, il.leaf_a, il.leaf_b, il.shift, st, mesh.leaf_start,
                                mesh.leaf_end, 1.0, pshift=p.image_shift)
    own = p.ghost == 0
    assert_fp32_close(grav.values[own], g["grav"][own], absg[own], what="step gravity")
    f, e, _ = compute_hydro_accel(p, mesh, st, il, mode=EvalMode.RELAXED)
    hk = hydro_force_kernel(2 * p.smoothing.max())
    absh = oracle.eval_abs_sums(hk, il.leaf_a, il.leaf_b, il.shift, st, mesh.leaf_start,
                                mesh.leaf_end, 1.0, pshift=p.image_shift)
    assert_fp32_close(np.column_stack([f, e])[own], np.column_stack(
        [g["hydro_force"], g["hydro_edot"]])[own], absh[own, :4], what="step hydro")
    fh = corrected_interpolate(p, mesh, st, il, crk, g["interp_field"], mode=EvalMode.RELAXED)
    inner = own & gas & ~crk.fallback
    err = np.abs(fh - g["interp"])[inner] / np.abs(g["interp"][inner]).max()
    assert err.max() <= 1e-5, err.max()


def test_gpu_adapt_smoothing_bitwise(golden):
    """Exact neighbour counts make the h iteration identical to the reference."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import ChainingMesh
    from paper_2510_03557_b200.hydro import adapt_smoothing_length
    from paper_2510_03557_b200.lane import EvalMode
    g = golden("adapt")
    p = particle_set(g, "in_")
    mv = MeshView(g, "mesh_")
    mesh = ChainingMesh(box=BoxGeometry(1.0), bounds_lo=None, bounds_hi=None,
                        bin_count=mv.bin_count, bin_width=mv.bin_width,
                        periodic_axis=mv.periodic_axis, n_particles=p.n,
                        leaf_start=mv.leaf_start, leaf_end=mv.leaf_end, leaf_lo=mv.leaf_lo,
                        leaf_hi=mv.leaf_hi, leaf_level=mv.leaf_level.copy(),
                        leaf_ghost_only=mv.leaf_ghost_only, leaf_bin=mv.leaf_bin,
                        _bin_ptr=mv._bin_ptr, _bin_ids=mv._bin_ids)
    h = adapt_smoothing_length(p, mesh, lambda: p.state_matrix(5 / 3), 40, float(g["bin_width"]),
                               mode=EvalMode.DETERMINISTIC)
    np.testing.assert_array_equal(h, g["h_out"])


def test_gpu_adapt_smoothing_resident_bitwise(golden):
    """No alias ghosts: adapt_smoothing_length iterates on the device (test on
    the device, numpy update of the moving rows) and still returns the
    reference's h bit for bit."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import ChainingMesh
    from paper_2510_03557_b200.hydro import adapt_smoothing_length
    from paper_2510_03557_b200.lane import EvalMode
    g = golden("adapt_periodic")
    p = particle_set(g, "in_")
    assert not np.any(p.ghost_src >= 0)
    mv = MeshView(g, "mesh_")
    mesh = ChainingMesh(box=BoxGeometry(1.0), bounds_lo=None, bounds_hi=None,
                        bin_count=mv.bin_count, bin_width=mv.bin_width,
                        periodic_axis=mv.periodic_axis, n_particles=p.n,
                        leaf_start=mv.leaf_start, leaf_end=mv.leaf_end, leaf_lo=mv.leaf_lo,
                        leaf_hi=mv.leaf_hi, leaf_level=mv.leaf_level.copy(),
                        leaf_ghost_only=mv.leaf_ghost_only, leaf_bin=mv.leaf_bin,
                        _bin_ptr=mv._bin_ptr, _bin_ids=mv._bin_ids)
    h = adapt_smoothing_length(p, mesh, lambda: p.state_matrix(5 / 3), 40, float(g["bin_width"]),
                               mode=EvalMode.DETERMINISTIC)
    np.testing.assert_array_equal(h, g["h_out"])


def test_gpu_nonfinite_raises(golden):
    from paper_2510_03557_b200.cmtree import InteractionList
    from paper_2510_03557_b200.errors import KernelEvalError
    from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
    g = golden("lane")
    k = f"c{g['configs'][0]}_"
    st = g[k + "state"].copy()
    st[:, 6] = np.nan  # NaN masses poison every gravity term
    ker = make_kernel("gravity", float(g[k + "reach"]), float(g[k + "spacing"]))
    il = InteractionList(g[k + "la"], g[k + "lb"], ker.reach, 0, g[k + "ls"])
    with pytest.raises(KernelEvalError, match="non-finite partial in leaf pair"):
        eval_interaction_list(ker, il, st, MeshView(g, k + "mesh_"), mode=EvalMode.RELAXED)


def test_gpu_resident_force_step(golden, oracle):
    """hb_force_step (the benchmark hot path) reproduces the reference step:
    same reorder, exact counts, density/CRK/gravity/hydro within tolerance."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import InteractionList
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.kernels import hydro_force_kernel
    from paper_2510_03557_b200.resident import StepConfig, force_step
    g = golden("step")
    p = particle_set(g, "in_")
    cfg = StepConfig(box=BoxGeometry(1.0), bin_width=float(g["bin_width"]), max_leaf_size=256,
                     r_s=float(g["r_s"]), r_cut=float(g["r_cut"]), softening=float(g["eps"]),
                     bounds_lo=g["bounds_lo"], bounds_hi=g["bounds_hi"])
    out = force_step(p, cfg)
    np.testing.assert_array_equal(p.global_id, g["built_global_id"])
    np.testing.assert_array_equal(p.ghost_src, g["built_ghost_src"])
    assert out["n_entries"] == g["la"].shape[0]
    np.testing.assert_array_equal(out["ncount"], g["ncount"])
    gas = p.species == 1
    rel = np.abs(p.density - g["density"])[gas] / g["density"][gas]
    assert np.median(rel) <= 1e-6 and rel.max() <= 1e-5, rel.max()
    np.testing.assert_array_equal(out["crk_fallback"], g["crk_fallback"])
    ok = gas & (g["crk_m0"] > 0)
    relA = np.abs(out["crk_A"] - g["crk_A"])[ok] / np.abs(g["crk_A"][ok])
    assert np.median(relA) <= 1e-6 and np.quantile(relA, 0.999) <= 1e-5, relA.max()
    z = g["crk_m0"] == 0   # non-gas and ghost-only rows: the reference's A = 1, B = 0
    np.testing.assert_array_equal(out["crk_A"][z], g["crk_A"][z])
    np.testing.assert_array_equal(out["crk_B"][z], g["crk_B"][z])
    own = p.ghost == 0
    st = g["state_eos"]
    ms = MeshView(g, "mesh_")
    gk = short_range_gravity_kernel(ForceSplit(r_s=float(g["r_s"]), r_cut=float(g["r_cut"])),
                                    float(g["eps"]))
    absg = oracle.eval_abs_sums(gk, g["la"], g["lb"], g["ls"], st, ms.leaf_start, ms.leaf_end, 1.0,
                                pshift=g["built_image_shift"])
    assert_fp32_close(out["grav"][own], g["grav"][own], absg[own], what="resident gravity")
    hk = hydro_force_kernel(2 * p.smoothing.max())
    absh = oracle.eval_abs_sums(hk, g["la"], g["lb"], g["ls"], st, ms.leaf_start, ms.leaf_end, 1.0,
                                pshift=g["built_image_shift"])
    ref_h = np.column_stack([g["hydro_force"], g["hydro_edot"]])
    assert_fp32_close(out["hydro"][own, :4], ref_h[own], absh[own, :4], what="resident hydro")


@pytest.mark.parametrize("sigma,h_jitter,mode,L,phys", [
    (0.05, 0.0, 0, 1.0, None), (1.0, 0.0, 0, 1.0, None), (2.5, 0.0, 0, 1.0, None),
    (1.0, 0.35, 0, 1.0, None), (1.0, 0.35, 1, 1.0, None), (1.0, 0.35, 0, 3.0, None),
    (1.0, 0.35, 0, 1.0, (1.4, 0.5, 1.0)), (1.0, 0.35, 1, 1.0, "leaf64")])
def test_gpu_force_step_vs_oracle_c1(oracle, sigma, h_jitter, mode, L, phys, monkeypatch):
    """hb_force_step at 2x32^3 (config C1, near-uniform and shell-crossing
    Zel'dovich ICs) against the oracle's ordered evaluation of the same step:
    leaf order and neighbour counts bit-exact, the rest within FP32 tolerance.
    h_jitter > 0: gas smoothing lengths scattered by +-h_jitter (adapted h
    varies between neighbours; the tile culls must use the tile's largest h).
    mode: HbStepArgs.gravity_mode -- 0 the default (bin tiles); 1 leaf tiles for
    gravity and SPH (the fallback when a bin outgrows the tiler).  L: box side
    (every length scales with it).  phys: (eos_gamma, visc_alpha, visc_beta)
    other than the defaults (5/3, 1, 2)."""
    max_leaf = 64 if phys == "leaf64" else 256     # "leaf64": leaves of <= 64
    gamma, alpha, beta = phys if isinstance(phys, tuple) else (5 / 3, 1.0, 2.0)
    monkeypatch.setenv("HB_GRAVITY_MODE", str(mode))
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.kernels import (crk_moments_kernel, density_kernel,
                                               hydro_force_kernel, neighbor_count_kernel)
    from paper_2510_03557_b200.resident import StepConfig, force_step
    npd = 32
    box = BoxGeometry(L)
    p0 = make_zeldovich_ic(npd, box, sigma)
    if h_jitter > 0:
        g0 = p0.species == 1
        rng = np.random.default_rng(17)
        p0.smoothing[g0] *= rng.uniform(1 - h_jitter, 1 + h_jitter, int(g0.sum()))
    pm = L / (2 * npd)
    r_s, r_cut = 2 * pm, 10 * pm
    eps = (L / p0.n ** (1 / 3)) / 50
    h_max = float(p0.smoothing.max())
    reach = max(r_cut, 2 * h_max)
    bw = max(4 * pm, reach * (1 + 1e-9))
    cfg = StepConfig(box=box, bin_width=bw, max_leaf_size=max_leaf, r_s=r_s, r_cut=r_cut,
                     softening=eps, eos_gamma=gamma, visc_alpha=alpha, visc_beta=beta)
    p = p0.copy()
    out = force_step(p, cfg)
    m = oracle.build_mesh(p0.pos, p0.image_shift, p0.ghost, L, bw, max_leaf)
    perm = m["perm"]
    np.testing.assert_array_equal(p.global_id, p0.global_id[perm])
    la, lb, ls = oracle.assemble(m, L, reach)
    assert out["n_entries"] == la.shape[0]
    q = p0.select(perm)
    st = q.state_matrix(gamma)
    args = (la, lb, ls, st, m["leaf_start"], m["leaf_end"], L)
    nc, _, _, _ = oracle.eval_pairs(neighbor_count_kernel(2 * h_max), *args, mode="deterministic",
                                    workers=8)
    np.testing.assert_array_equal(out["ncount"], nc[:, 0])
    dk = density_kernel(2 * h_max)
    rho, _, _, _ = oracle.eval_pairs(dk, *args, mode="relaxed", workers=8)
    gas = q.species == 1
    rel = np.abs(p.density - rho[:, 0])[gas] / rho[gas, 0]
    assert np.median(rel) <= 1e-6 and np.quantile(rel, 0.999) <= 1e-5, rel.max()
    q.density[gas] = rho[gas, 0]
    oracle.refresh_eos(st, q.density, q.internal_energy, gamma)
    ck = crk_moments_kernel(2 * h_max)
    mom, _, _, _ = oracle.eval_pairs(ck, *args, mode="relaxed", workers=8)
    mabs = oracle.eval_abs_sums(ck, *args)
    assert_fp32_close(out["crk_moments"], mom, mabs, what="crk moments")
    A, B, fb, *_ = oracle.crk_solve(mom, gas)
    np.testing.assert_array_equal(out["crk_fallback"], fb)
    relA = np.abs(out["crk_A"] - A)[gas] / np.abs(A[gas])
    assert np.median(relA) <= 1e-5 and np.quantile(relA, 0.999) <= 1e-4, relA.max()
    gk = short_range_gravity_kernel(ForceSplit(r_s=r_s, r_cut=r_cut), eps)
    g, _, _, _ = oracle.eval_pairs(gk, *args, mode="relaxed", workers=8)
    gabs = oracle.eval_abs_sums(gk, *args)
    assert_fp32_close(out["grav"], g, gabs, what="gravity")
    hk = hydro_force_kernel(2 * h_max, alpha, beta)
    hy, _, _, _ = oracle.eval_pairs(hk, *args, mode="relaxed", workers=8)
    habs = oracle.eval_abs_sums(hk, *args)
    assert_fp32_close(out["hydro"], hy, habs, what="hydro")


def test_gpu_host_stepper_matches_sync_step(golden):
    """The e2e path (HostStepper: pinned H2D, step with deferred status, D2H
    queued before the host waits) returns what the synchronous step returns."""
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.resident import STEP_FIELDS, HostStepper, ResidentRank, StepConfig
    g = golden("step")
    cfg = StepConfig(box=BoxGeometry(1.0), bin_width=float(g["bin_width"]), max_leaf_size=256,
                     r_s=float(g["r_s"]), r_cut=float(g["r_cut"]), softening=float(g["eps"]),
                     bounds_lo=g["bounds_lo"], bounds_hi=g["bounds_hi"])
    p = particle_set(g, "in_")
    ref = ResidentRank(p.copy(), cfg)
    ref_out = {k: v.cpu().numpy() for k, v in ref.step().items()}
    ref_density = ref.fields()["density"].cpu().numpy()
    ref_fields = {f: v.cpu().numpy() for f, v in ref.fields().items()}
    rk = ResidentRank(p.copy(), cfg)
    pin_in = {f: torch.from_numpy(np.ascontiguousarray(getattr(p, f))).pin_memory()
              for f in STEP_FIELDS}
    names = ("grav", "hydro", "ncount", "crk_A", "crk_B", "perm")
    pin_out = {k: torch.empty(rk.out[k].shape, dtype=rk.out[k].dtype).pin_memory() for k in names}
    pin_out["density"] = torch.empty(rk.n, dtype=torch.float64).pin_memory()
    hs = HostStepper(rk, pin_in, pin_out)
    for _ in range(2):   # the second call reuses the buffers and the status word
        got = {k: v.numpy().copy() for k, v in hs().items()}
        np.testing.assert_array_equal(got["perm"][:p.n], ref_out["perm"][:p.n])
        np.testing.assert_array_equal(got["ncount"][:p.n], ref_out["ncount"][:p.n])
        for k in ("grav", "hydro", "crk_A", "crk_B"):
            np.testing.assert_allclose(got[k][:p.n], ref_out[k][:p.n], rtol=1e-6, atol=1e-12,
                                       err_msg=k)
        np.testing.assert_allclose(got["density"], ref_density, rtol=1e-6)
        for f, v in rk.fields().items():   # the split (early / late) gather
            np.testing.assert_array_equal(v.cpu().numpy(), ref_fields[f], err_msg=f)


def test_gpu_resident_nonfinite_raises_sync_and_deferred(golden):
    """A non-finite partial stops the resident step with the reference's error
    (KernelEvalError), both from the synchronous call and from HostStepper's
    deferred status check."""
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.errors import HydroboxError
    from paper_2510_03557_b200.resident import STEP_FIELDS, HostStepper, ResidentRank, StepConfig
    g = golden("step")
    cfg = StepConfig(box=BoxGeometry(1.0), bin_width=float(g["bin_width"]), max_leaf_size=256,
                     r_s=float(g["r_s"]), r_cut=float(g["r_cut"]), softening=float(g["eps"]),
                     bounds_lo=g["bounds_lo"], bounds_hi=g["bounds_hi"])
    p = particle_set(g, "in_")
    p.mass[np.nonzero(p.ghost == 0)[0][7]] = np.inf
    with pytest.raises(HydroboxError):
        ResidentRank(p.copy(), cfg).step()
    rk = ResidentRank(p.copy(), cfg)
    pin_in = {f: torch.from_numpy(np.ascontiguousarray(getattr(p, f))).pin_memory()
              for f in STEP_FIELDS}
    names = ("grav", "hydro", "ncount", "crk_A", "crk_B", "perm")
    pin_out = {k: torch.empty(rk.out[k].shape, dtype=rk.out[k].dtype).pin_memory() for k in names}
    pin_out["density"] = torch.empty(rk.n, dtype=torch.float64).pin_memory()
    with pytest.raises(HydroboxError):
        HostStepper(rk, pin_in, pin_out)()


def test_gpu_host_stepper_four_groups_matches_sync_step():
    """A set without ghost rows takes HostStepper's four-group upload (density,
    ids and ghost sources land while pass B runs, HbStepArgs.last_fields_event):
    every output and every reordered field equals the synchronous step's."""
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.resident import STEP_FIELDS, HostStepper, ResidentRank, StepConfig
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(20, box, 1.0)
    p.density[:] = np.linspace(0.5, 1.5, p.n)   # input densities: the DM rows keep theirs
    d = 1.0 / 20
    reach = max(5 * d, 2 * float(p.smoothing.max()))
    cfg = StepConfig(box=box, bin_width=reach * (1 + 1e-9), max_leaf_size=256, r_s=d,
                     r_cut=5 * d, softening=(1.0 / p.n ** (1 / 3)) / 50)
    ref = ResidentRank(p.copy(), cfg)
    ref_out = {k: v[:p.n].cpu().numpy().copy() for k, v in ref.step().items()}
    ref_fields = {f: v.cpu().numpy().copy() for f, v in ref.fields().items()}
    rk = ResidentRank(p.copy(), cfg)
    pin_in = {f: torch.from_numpy(np.ascontiguousarray(getattr(p, f))).pin_memory()
              for f in STEP_FIELDS}
    names = ("grav", "hydro", "ncount", "crk_A", "crk_B", "perm")
    pin_out = {k: torch.empty(rk.out[k].shape, dtype=rk.out[k].dtype).pin_memory() for k in names}
    pin_out["density"] = torch.empty(rk.n, dtype=torch.float64).pin_memory()
    hs = HostStepper(rk, pin_in, pin_out)
    assert hs.four_groups
    for _ in range(2):
        got = {k: v.numpy().copy() for k, v in hs().items()}
        for k in names:
            np.testing.assert_array_equal(got[k][:p.n], ref_out[k], err_msg=k)
        np.testing.assert_array_equal(got["density"], ref_fields["density"])
        for f, v in rk.fields().items():
            np.testing.assert_array_equal(v.cpu().numpy(), ref_fields[f], err_msg=f)


def test_gpu_last_fields_event_rejects_ghost_rows(golden):
    """The four-group upload (HbStepArgs.last_fields_event) is only for sets
    without ghost rows; on an overloaded set the step raises HydroboxError."""
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.errors import HydroboxError
    from paper_2510_03557_b200.resident import ResidentRank, StepConfig
    g = golden("step")
    cfg = StepConfig(box=BoxGeometry(1.0), bin_width=float(g["bin_width"]), max_leaf_size=256,
                     r_s=float(g["r_s"]), r_cut=float(g["r_cut"]), softening=float(g["eps"]),
                     bounds_lo=g["bounds_lo"], bounds_hi=g["bounds_hi"])
    p = particle_set(g, "in_")
    assert np.any(p.ghost)
    rk = ResidentRank(p, cfg)
    ev_late, ev_last = torch.cuda.Event(), torch.cuda.Event()
    ev_late.record()
    ev_last.record()
    with pytest.raises(HydroboxError, match="ghost rows"):
        rk.step(late_fields=ev_late, last_fields=ev_last)


def test_gpu_removed_gravity_modes_raise():
    """HbStepArgs.gravity_mode 2 / 3 (round 1's half-warp and r/t-table
    variants) were removed: the step says so instead of silently running
    something else."""
    import os
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.errors import HydroboxError
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.resident import ResidentRank, StepConfig
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(12, box, 0.5)
    d = 1.0 / 12
    cfg = StepConfig(box=box, bin_width=max(5 * d, 2 * float(p.smoothing.max())) * (1 + 1e-9),
                     max_leaf_size=256, r_s=d, r_cut=5 * d, softening=d / 60)
    old = os.environ.get("HB_GRAVITY_MODE")
    try:
        os.environ["HB_GRAVITY_MODE"] = "2"
        with pytest.raises(HydroboxError, match="removed"):
            ResidentRank(p, cfg).step()
    finally:
        if old is None:
            os.environ.pop("HB_GRAVITY_MODE", None)
        else:
            os.environ["HB_GRAVITY_MODE"] = old
