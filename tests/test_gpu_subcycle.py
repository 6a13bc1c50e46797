"""Hierarchical subcycle integrator against the
reference's subcycle_pm_step (hb/stepper.py:103-192) on the golden periodic
2x8^3 interval (tests/golden/subcycle.npz, made by tests/golden/make_golden.py).

Bit-exact: the per-boundary (s, depth, level, unordered due pairs) log, and the
deterministic momentum audit (sum of impulse quanta = 0 at every boundary).
FP32 tolerance: the velocity and internal-energy CHANGES over the interval (the
impulses; the totals are dominated by the unchanged initial values), density,
the recorded short-range acceleration, positions and grown leaf boxes."""
import numpy as np
import pytest

from tests.conftest import MeshView

pytestmark = pytest.mark.gpu


def _inputs(g):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.particles import ParticleSet
    n = g["in_pos"].shape[0]
    p = ParticleSet(n)
    for k in ("pos", "vel", "mass", "smoothing", "internal_energy", "density", "species",
              "ghost", "image_shift", "global_id", "ghost_src", "timestep_level"):
        getattr(p, k)[...] = g["in_" + k]
    p.accel[...] = g["in_accel"]
    return p, MeshView(g, "mesh_"), BoxGeometry(1.0)


def _norm_err(ours, ref):
    """max |ours - ref| over the rms of ref (per-component arrays)."""
    scale = np.sqrt(np.mean(ref ** 2)) + 1e-300
    return float(np.max(np.abs(ours - ref)) / scale)


@pytest.mark.parametrize("tag", ["det", "rel"])
def test_subcycle_matches_reference(golden, tag):
    from paper_2510_03557_b200.hydro import TimestepHierarchy
    from paper_2510_03557_b200.kernels import gravity_kernel
    from paper_2510_03557_b200.lane import EvalMode
    from paper_2510_03557_b200.stepper import ShortRangeContext, subcycle_pm_step
    g = golden("subcycle")
    p, mesh, box = _inputs(g)
    mode = EvalMode.DETERMINISTIC if tag == "det" else EvalMode.RELAXED
    hier = TimestepHierarchy(dt_pm=float(g["dt_pm"]), max_level=int(g["max_level"]),
                             n_levels=int(g["n_levels"]))
    ctx = ShortRangeContext(particles=p, mesh=mesh, box=box, eos_gamma=5 / 3,
                            reach=float(g["reach"]), mode=mode,
                            gravity_kernel=gravity_kernel(float(g["r_s"]), float(g["r_cut"]),
                                                          float(g["eps"])),
                            hydro_enabled=True)
    audit = subcycle_pm_step(ctx, hier)
    log = np.array([(r.s, r.depth, lv, n) for r in audit.boundary_log
                    for lv, n in sorted(r.pairs_per_level.items())], dtype=np.int64)
    np.testing.assert_array_equal(log, g[f"{tag}_pairs_log"])
    assert audit.n_boundaries == hier.n_fine + 1
    assert audit.max_momentum_quanta == 0 == int(g[f"{tag}_max_quanta"])
    dv, dv_ref = p.vel - g["in_vel"], g[f"{tag}_vel"] - g["in_vel"]
    du, du_ref = (p.internal_energy - g["in_internal_energy"],
                  g[f"{tag}_internal_energy"] - g["in_internal_energy"])
    gas = g["in_species"] == 1
    assert _norm_err(dv, dv_ref) <= 2e-4, _norm_err(dv, dv_ref)
    assert _norm_err(du[gas], du_ref[gas]) <= 2e-4, _norm_err(du[gas], du_ref[gas])
    assert _norm_err(p.accel, g[f"{tag}_accel"]) <= 2e-4
    np.testing.assert_allclose(p.density[gas], g[f"{tag}_density"][gas], rtol=1e-5)
    np.testing.assert_allclose(p.pos, g[f"{tag}_pos"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(mesh.leaf_lo, g[f"{tag}_leaf_lo"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(mesh.leaf_hi, g[f"{tag}_leaf_hi"], rtol=0, atol=1e-10)
