"""GPU, at the benchmark's full size (c2: 2x128^3, z=10 Zel'dovich): properties
that hold at any size, where the oracle is too slow to compare directly.

* the step's permutation is a bijection, and the reordered fields are the
  inputs permuted, bit for bit;
* two steps on the same input are bitwise identical (deterministic gather);
* pairwise antisymmetry: total gravity and hydro force cancel (sum m a ~ 0
  relative to sum |m a|, FP32 pair sums);
* neighbour counts are integers near the lattice mean 4/3 pi (2.6)^3 + 1;
* SPH densities equal the mean gas density 1/2 to within a few per cent on
  this near-uniform lattice, and CRK needs no fallback."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2_steps():
    import bench
    from paper_2510_03557_b200.resident import STEP_FIELDS, ResidentRank
    p, cfg, meta = bench.make_workload("c2")
    inputs = {f: np.array(getattr(p, f), copy=True) for f in STEP_FIELDS}
    outs = []
    for _ in range(2):
        rk = ResidentRank(p.copy(), cfg)
        out = {k: v.cpu().numpy() for k, v in rk.step().items()}
        fields = {f: v.cpu().numpy() for f, v in rk.fields().items()}
        outs.append((out, fields))
    return p, inputs, outs


def test_permutation_and_reorder_exact(c2_steps):
    p, inputs, outs = c2_steps
    out, fields = outs[0]
    perm = out["perm"][:p.n]
    assert np.array_equal(np.sort(perm), np.arange(p.n))
    for f, v in inputs.items():
        if f in ("density", "ghost_src"):
            continue   # density is recomputed; ghost_src is remapped through the permutation
        np.testing.assert_array_equal(fields[f], v[perm], err_msg=f)


def test_deterministic(c2_steps):
    _, _, ((o1, f1), (o2, f2)) = c2_steps
    for k in o1:
        np.testing.assert_array_equal(o1[k], o2[k], err_msg=k)
    for k in f1:
        np.testing.assert_array_equal(f1[k], f2[k], err_msg=k)


def test_forces_cancel(c2_steps):
    p, _, ((out, _), _) = c2_steps
    g = out["grav"][:p.n]
    assert np.abs(g.sum(0)).max() <= 1e-5 * np.abs(g).sum(0).max()
    h = out["hydro"][:p.n, :3]
    assert np.abs(h.sum(0)).max() <= 1e-5 * np.abs(h).sum(0).max()


def test_counts_density_crk(c2_steps):
    p, _, ((out, fields), _) = c2_steps
    gas = fields["species"] == 1
    nc = out["ncount"][:p.n][gas]
    assert np.array_equal(nc, np.round(nc))
    mean_expected = 4.0 / 3.0 * math.pi * 2.6 ** 3 + 1   # gas per d^3 = 1, self included
    assert abs(nc.mean() / mean_expected - 1) < 0.1, nc.mean()
    rho = fields["density"][gas]
    assert np.all(rho > 0)
    assert abs(np.median(rho) / 0.5 - 1) < 0.03, np.median(rho)
    assert not out["crk_fallback"][:p.n][gas].any()


def test_restep_after_motion_matches_fresh():
    """A resident rank stepped again after its particles moved (the simulation
    loop: buffers flip, the mesh is rebuilt from the previous leaf order)
    gives, per global id, what a fresh rank gives on the moved set."""
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.particles import ParticleSet
    from paper_2510_03557_b200.resident import STEP_FIELDS, ResidentRank, StepConfig
    box = BoxGeometry(1.0)
    npd = 32
    p = make_zeldovich_ic(npd, box, 0.5)
    pm = 1.0 / (2 * npd)
    cfg = StepConfig(box=box, bin_width=10 * pm * (1 + 1e-9), max_leaf_size=256, r_s=2 * pm,
                     r_cut=10 * pm, softening=(1.0 / p.n ** (1 / 3)) / 50)
    rk = ResidentRank(p.copy(), cfg)
    rk.step()
    f = rk.fields()
    g = torch.Generator(device="cuda").manual_seed(5)
    f["pos"] += (torch.rand(f["pos"].shape, generator=g, device="cuda",
                            dtype=torch.float64) - 0.5) * (0.8 / npd)
    f["pos"].remainder_(1.0)
    moved = ParticleSet(p.n)
    for k in STEP_FIELDS:
        setattr(moved, k, f[k].cpu().numpy().copy())
    out2 = {k: v.cpu().numpy() for k, v in rk.step().items()}
    gid2 = rk.fields()["global_id"].cpu().numpy()
    fresh = ResidentRank(moved, cfg)
    out_f = {k: v.cpu().numpy() for k, v in fresh.step().items()}
    gid_f = fresh.fields()["global_id"].cpu().numpy()
    a, b = np.argsort(gid2), np.argsort(gid_f)
    np.testing.assert_array_equal(out2["ncount"][a], out_f["ncount"][b])
    for k in ("grav", "hydro", "crk_A"):   # FP32 sums, possibly in another order
        x, y = out2[k][a], out_f[k][b]
        scale = np.abs(y).max()
        err = np.abs(x - y).reshape(len(x), -1).max(axis=1)
        assert err.max() <= 1e-4 * scale, (k, err.max() / scale)
        assert np.median(err) <= 1e-6 * scale, (k, np.median(err) / scale)
