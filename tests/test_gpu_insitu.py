"""In-situ cluster finding against the reference's
hb/insitu.py on the golden clustered box (tests/golden/fof.npz): FOF and DBSCAN
on one periodic set and on (2,2,1) overloaded rank sets (global-id stitching).
Bit-exact: group memberships, halo ids, counts, DBSCAN noise.  rtol 1e-12:
masses, centres, radii.  P(k) of the CIC density (cuFFT): rtol 1e-10."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _set(g, prefix=""):
    from paper_2510_03557_b200.particles import ParticleSet
    n = g[prefix + "pos"].shape[0]
    p = ParticleSet(n)
    for k in ("pos", "mass", "global_id", "species") + (
            ("vel", "smoothing", "internal_energy", "density", "ghost", "image_shift",
             "ghost_src") if prefix else ()):
        getattr(p, k)[...] = g[prefix + k]
    return p


def _check(groups, g, tag):
    np.testing.assert_array_equal([q.halo_id for q in groups], g[f"{tag}_halo_id"])
    np.testing.assert_array_equal([q.count for q in groups], g[f"{tag}_count"])
    members = np.concatenate([q.member_ids for q in groups]) if groups else np.zeros(0)
    np.testing.assert_array_equal(members, g[f"{tag}_members"])
    np.testing.assert_allclose([q.total_mass for q in groups], g[f"{tag}_mass"], rtol=1e-12)
    np.testing.assert_allclose(np.array([q.center for q in groups]).reshape(-1, 3),
                               g[f"{tag}_center"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose([q.radius for q in groups], g[f"{tag}_radius"], rtol=1e-12,
                               atol=1e-14)


def test_fof_dbscan_match_reference(golden):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.insitu import dbscan_find, fof_find
    g = golden("fof")
    box = BoxGeometry(1.0)
    p = _set(g)
    sets = [_set(g, f"rank{r}_") for r in range(4)]
    ll, eps, w = float(g["ll"]), float(g["eps"]), float(g["w"])
    _check(fof_find(p, box, ll, min_members=5), g, "fof1")
    _check(fof_find(sets, box, ll, min_members=5, overload_width=w), g, "fof4")
    g1, n1 = dbscan_find(p, box, eps, 6)
    _check(g1, g, "db1")
    np.testing.assert_array_equal(n1, g["db1_noise"])
    g4, n4 = dbscan_find(sets, box, eps, 6, overload_width=w)
    _check(g4, g, "db4")
    np.testing.assert_array_equal(n4, g["db4_noise"])


def test_power_spectrum_matches_reference(golden):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.insitu import power_spectrum
    g = golden("fof")
    k, pk, cnt = power_spectrum(g["pk_rho"], BoxGeometry(1.0))
    np.testing.assert_array_equal(cnt, g["pk_counts"])
    np.testing.assert_allclose(k, g["pk_k"], rtol=1e-15)
    np.testing.assert_allclose(pk, g["pk"], rtol=1e-10, atol=1e-14 * np.abs(g["pk"]).max())
