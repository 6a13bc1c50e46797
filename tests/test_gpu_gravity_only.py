"""GPU: the pieces of the gravity-only (dark-matter) configs.

* make_zeldovich_ic_device (cuFFT displacement field, device-side selection)
  returns the rows make_zeldovich_ic(select=...) returns: same particles and
  ids, positions and velocities equal to FFT rounding;
* a gravity_only ResidentRank (no SPH buffers) gives bitwise the gravity of a
  full rank run with PASS_GRAVITY."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("species", ["both", "dm"])
def test_device_ic_matches_numpy(species):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.distributed import rank_grid_for
    from paper_2510_03557_b200.domain import owner_ranks, owner_ranks_torch
    from paper_2510_03557_b200.ic import make_zeldovich_ic, make_zeldovich_ic_device
    box = BoxGeometry(1.0)
    grid = rank_grid_for(4)
    for r in (0, 3):
        ref = make_zeldovich_ic(32, box, 0.3, species=species,
                                select=lambda pos: owner_ranks(pos, box, grid) == r)
        got = make_zeldovich_ic_device(32, box, 0.3,
                                       lambda pos: owner_ranks_torch(pos, box, grid) == r,
                                       species=species)
        np.testing.assert_array_equal(got.global_id, ref.global_id)
        np.testing.assert_allclose(got.pos, ref.pos, rtol=0, atol=1e-13)
        np.testing.assert_allclose(got.vel, ref.vel, rtol=0, atol=1e-14)
        for f in ("mass", "smoothing", "internal_energy", "species"):
            np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f)


def test_gravity_only_rank_equals_full_rank_gravity():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.resident import PASS_GRAVITY, ResidentRank, StepConfig
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(32, box, 0.3, species="dm")
    r_s = 1.0 / 32
    cfg = StepConfig(box=box, bin_width=5 * r_s * (1 + 1e-9), max_leaf_size=256, r_s=r_s,
                     r_cut=5 * r_s, softening=(1.0 / 32) / 50)
    full = ResidentRank(p.copy(), cfg)
    g_full = full.step(PASS_GRAVITY)["grav"].cpu().numpy()
    lean = ResidentRank(p.copy(), cfg, gravity_only=True)
    out = lean.step(PASS_GRAVITY)
    assert set(out) == {"perm", "grav"}
    np.testing.assert_array_equal(out["grav"].cpu().numpy(), g_full)
    np.testing.assert_array_equal(out["perm"].cpu().numpy(), full.out["perm"].cpu().numpy())
    assert np.abs(g_full).max() > 0
