"""CPU: the sampled-receiver oracle (tests/_parity.py) that the full-size GPU
parity tests rely on returns, on its sampled rows, exactly what the oracle's
evaluation of the whole list returns (compaction and entry selection change
nothing a receiver sees)."""
import numpy as np


def test_sampled_oracle_equals_full_oracle(oracle):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.kernels import crk_moments_kernel, hydro_force_kernel
    from paper_2510_03557_b200.resident import StepConfig
    from tests._parity import SampledOracle
    box = BoxGeometry(1.0)
    npd = 16
    p = make_zeldovich_ic(npd, box, 1.0)
    d = 1.0 / npd
    r_s, r_cut = d, 5 * d
    h = float(p.smoothing.max())
    reach = max(r_cut, 2 * h)
    cfg = StepConfig(box=box, bin_width=reach * (1 + 1e-9), max_leaf_size=64, r_s=r_s,
                     r_cut=r_cut, softening=(1.0 / p.n ** (1 / 3)) / 50)
    so = SampledOracle(oracle, p, cfg, stride=5, crowded_bins=2, workers=1)
    assert 0 < so.recv.size < so.rows.size <= p.n
    # the whole list on the whole (leaf-ordered) set
    m = so.mesh
    la, lb, ls = oracle.assemble(m, 1.0, reach)
    assert la.shape[0] == so.n_entries
    q = p.select(m["perm"])
    st = q.state_matrix(cfg.eos_gamma)
    args = (la, lb, ls, st, m["leaf_start"], m["leaf_end"], 1.0)
    rows = so.rows[so.recv]
    gk = short_range_gravity_kernel(ForceSplit(r_s=r_s, r_cut=r_cut), cfg.softening)
    g_full, _, _, _ = oracle.eval_pairs(gk, *args, mode="relaxed", workers=1)
    g, gabs, _ = so.gravity()
    np.testing.assert_array_equal(g[so.recv], g_full[rows])
    ab_full = oracle.eval_abs_sums(gk, *args, workers=1)
    np.testing.assert_array_equal(gabs[so.recv], ab_full[rows])
    nc, rho = so.counts_density()
    from paper_2510_03557_b200.kernels import density_kernel, neighbor_count_kernel
    nc_full, _, _, _ = oracle.eval_pairs(neighbor_count_kernel(2 * h), *args, mode="deterministic")
    np.testing.assert_array_equal(nc[so.recv], nc_full[rows, 0])
    rho_full, _, _, _ = oracle.eval_pairs(density_kernel(2 * h), *args, mode="relaxed", workers=1)
    np.testing.assert_array_equal(rho[so.recv], rho_full[rows, 0])
    # CRK / hydro on a given density field (the GPU's, in the real test)
    dens = np.where(q.species == 1, rho_full[:, 0], q.density)
    mom, mabs, A, B, fb = so.crk(dens[so.rows])
    st2 = st.copy()
    oracle.refresh_eos(st2, dens, q.internal_energy, cfg.eos_gamma)
    mom_full, _, _, _ = oracle.eval_pairs(crk_moments_kernel(2 * h), *args[:3], st2, *args[4:],
                                          mode="relaxed", workers=1)
    np.testing.assert_array_equal(mom[so.recv], mom_full[rows])
    hy, _ = so.hydro(dens[so.rows])
    hy_full, _, _, _ = oracle.eval_pairs(hydro_force_kernel(2 * h), *args[:3], st2, *args[4:],
                                         mode="relaxed", workers=1)
    np.testing.assert_array_equal(hy[so.recv], hy_full[rows])
