"""PM long-range gravity against the reference's
hb/gravity.py pipeline (fixture tests/golden/pm.npz from tests/golden/make_golden.py),
plus size-independent properties: total long-range momentum cancels and a lone
particle feels no self-force (matched deposit / gather stencils, real even D(k)).

Tolerances (float64 throughout; the differences are atomic-add order in the
deposit and cuFFT vs pocketfft rounding): deposit rtol 1e-12, influence rtol
1e-10, fields / potential / accelerations within 1e-10 of their max."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _close(ours, ref, rel):
    scale = float(np.max(np.abs(ref))) + 1e-300
    assert float(np.max(np.abs(ours - ref))) <= rel * scale, (
        float(np.max(np.abs(ours - ref))) / scale)


@pytest.mark.parametrize("fixture", ["pm", "pm_L2"])
def test_pm_matches_reference(golden, fixture):
    from paper_2510_03557_b200 import gravity as G
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.particles import ParticleSet
    g = golden(fixture)
    L = float(g["L"]) if "L" in g else 1.0
    box = BoxGeometry(L)
    p = ParticleSet(g["pos"].shape[0])
    p.pos[...] = g["pos"]
    p.mass[...] = g["mass"]
    n = int(g["grid_n"])
    split = G.ForceSplit(r_s=float(g["r_s"]), r_cut=float(g["r_cut"]))
    rho = G.deposit_cic(p, n, box)
    np.testing.assert_allclose(rho.values, g["rho"], rtol=1e-12, atol=1e-12 * g["rho"].max())
    h3 = (L / n) ** 3
    assert abs(rho.values.sum() * h3 - p.mass.sum()) <= 1e-12 * p.mass.sum()
    d = G.optimal_influence_device(n, box, split.r_s).cpu().numpy()
    np.testing.assert_allclose(d, g["d_opt"], rtol=1e-10, atol=1e-12 * np.abs(g["d_opt"]).max())
    for tag in ("optimal", "naive"):
        fields, pot = G.solve_long_range(rho, split, box, want_potential=True, influence=tag)
        _close(np.stack([f.values for f in fields]), g[f"{tag}_fields"], 1e-10)
        _close(pot.values, g[f"{tag}_pot"], 1e-10)
        acc = G.interpolate_force(fields, p)
        _close(acc, g[f"{tag}_acc"], 1e-10)
        e = G.long_range_potential_energy(pot, p)
        assert math.isclose(e, float(g[f"{tag}_energy"]), rel_tol=1e-10)


def test_pm_momentum_and_self_force():
    import torch
    from paper_2510_03557_b200 import gravity as G
    from paper_2510_03557_b200.box import BoxGeometry
    box = BoxGeometry(1.0)
    n = 64
    solver = G.LongRangeSolver(n, G.ForceSplit.for_grid(box, n), box)
    rng = np.random.default_rng(8)
    pos = torch.from_numpy(rng.random((200_000, 3))).cuda()
    mass = torch.from_numpy(rng.uniform(0.5, 1.5, 200_000) / 200_000).cuda()
    acc, phi = solver.accelerations(pos, mass, want_potential=True)
    mom = (acc * mass[:, None]).sum(dim=0).abs().max().item()
    scale = (acc.abs() * mass[:, None]).sum().item()
    assert mom <= 1e-10 * scale, mom / scale
    # one particle: its own long-range force vanishes at any position
    for x in rng.random((5, 3)):
        one = torch.from_numpy(x[None, :]).cuda()
        a1, _ = solver.accelerations(one, torch.ones(1, dtype=torch.float64, device="cuda"))
        assert a1.abs().max().item() <= 1e-9, a1
