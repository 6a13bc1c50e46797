"""CPU: the C oracle restatement is pinned bitwise to the reference's own
outputs (golden vectors from tests/golden/make_golden.py)."""
import numpy as np
import pytest

from paper_2510_03557_b200 import kernels as KK
from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel

KERNELS = ["counting", "gravity", "grav_pot", "density", "neighbor_count", "crk_moments", "hydro",
           "crk_interp"]


def make_kernel(name, reach, spacing):
    if name == "counting":
        return KK.counting_kernel(reach)
    if name == "gravity":
        return short_range_gravity_kernel(ForceSplit(r_s=reach / 5.0, r_cut=reach), spacing / 50)
    if name == "grav_pot":
        return KK.gravity_potential_kernel(reach / 5.0, reach, spacing / 50)
    if name == "density":
        return KK.density_kernel(reach)
    if name == "neighbor_count":
        return KK.neighbor_count_kernel(reach)
    if name == "crk_moments":
        return KK.crk_moments_kernel(reach)
    if name == "hydro":
        return KK.hydro_force_kernel(reach)
    if name == "crk_interp":
        return KK.crk_interp_kernel(reach)
    raise KeyError(name)


@pytest.mark.parametrize("name", KERNELS)
def test_lane_core_bitwise(golden, oracle, name):
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        st = g[k + "state"]
        ker = make_kernel(name, float(g[k + "reach"]), float(g[k + "spacing"]))
        aux = g[k + "aux"] if ker.n_aux else None
        for mode, tag in (("relaxed", "rel"), ("deterministic", "det")):
            vals, iacc, cnt, err = oracle.eval_pairs(
                ker, g[k + "la"], g[k + "lb"], g[k + "ls"], st, g[k + "mesh_leaf_start"],
                g[k + "mesh_leaf_end"], 1.0, mode=mode, workers=1, aux=aux)
            assert err == 0
            np.testing.assert_array_equal(vals, g[k + f"{name}_{tag}"])
            ref_c = g[k + f"{name}_{tag}_counters"]
            got_c = [cnt[x] for x in ("f_evals", "g_evals", "rotations", "pairs_scheduled",
                                      "pairs_in_reach")]
            np.testing.assert_array_equal(got_c, ref_c)
            if tag == "det":
                np.testing.assert_array_equal(iacc, g[k + f"{name}_detint"])


def test_worker_split_merge_order(golden, oracle):
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        ker = make_kernel("gravity", float(g[k + "reach"]), float(g[k + "spacing"]))
        vals, _, _, _ = oracle.eval_pairs(ker, g[k + "la"], g[k + "lb"], g[k + "ls"],
                                          g[k + "state"], g[k + "mesh_leaf_start"],
                                          g[k + "mesh_leaf_end"], 1.0, mode="relaxed", workers=3)
        np.testing.assert_array_equal(vals, g[k + "gravity_rel_w3"])


@pytest.mark.parametrize("name", ["gravity", "hydro"])
def test_mirror_bitwise(golden, oracle, name):
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        ker = make_kernel(name, float(g[k + "reach"]), float(g[k + "spacing"]))
        for mode, tag in (("relaxed", "rel"), ("deterministic", "det")):
            vals, _, _, _ = oracle.eval_pairs(ker, g[k + "ua"], g[k + "ub"], g[k + "us"],
                                              g[k + "state"], g[k + "mesh_leaf_start"],
                                              g[k + "mesh_leaf_end"], 1.0, mode=mode, mirror=True)
            np.testing.assert_array_equal(vals, g[k + f"{name}_mirror_{tag}"])


@pytest.mark.parametrize("name", KERNELS)
def test_allpairs_bitwise(golden, oracle, name):
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        ker = make_kernel(name, float(g[k + "reach"]), float(g[k + "spacing"]))
        aux = g[k + "aux"] if ker.n_aux else None
        vals, absum = oracle.reference_pair_sum(ker, g[k + "state"], 1.0, mode="relaxed", aux=aux)
        np.testing.assert_array_equal(vals, g[k + f"{name}_allpairs"])
        np.testing.assert_array_equal(absum, g[k + f"{name}_allpairs_abs"])


@pytest.mark.parametrize("case", ["rand", "lat", "clu", "r221"])
def test_mesh_and_lists_bitwise(golden, oracle, case):
    g = golden("mesh")
    k = case + "_"
    m = oracle.build_mesh(g[k + "in_pos"], g[k + "in_image_shift"], g[k + "in_ghost"], 1.0,
                          float(g[k + "bin_width"]), int(g[k + "max_leaf"]),
                          g[k + "bounds_lo"], g[k + "bounds_hi"])
    np.testing.assert_array_equal(g[k + "in_global_id"][m["perm"]], g[k + "out_global_id"])
    for f in ("leaf_start", "leaf_end", "leaf_lo", "leaf_hi", "leaf_ghost_only", "leaf_bin",
              "bin_count", "bin_width"):
        np.testing.assert_array_equal(m[f], g[k + "mesh_" + f], err_msg=f)
    np.testing.assert_array_equal(m["periodic"], g[k + "mesh_periodic"])
    np.testing.assert_array_equal(m["bin_ptr"], g[k + "mesh_bin_ptr"])
    ri = 0
    while k + f"list{ri}_a" in g:
        la, lb, ls = oracle.assemble(m, 1.0, float(g[k + f"list{ri}_reach"]), 0)
        np.testing.assert_array_equal(la, g[k + f"list{ri}_a"])
        np.testing.assert_array_equal(lb, g[k + f"list{ri}_b"])
        np.testing.assert_array_equal(ls, g[k + f"list{ri}_s"])
        ri += 1
    la, lb, ls = oracle.assemble(m, 1.0, float(g[k + "list0_reach"]), 1, leaf_level=g[k + "levels"])
    np.testing.assert_array_equal(la, g[k + "listd1_a"])
    np.testing.assert_array_equal(lb, g[k + "listd1_b"])
    np.testing.assert_array_equal(ls, g[k + "listd1_s"])


def test_step_crk_solve(golden, oracle):
    """moments -> A, B, fallback restatement vs compute_crk_coefficients."""
    g = golden("step")
    vals = np.zeros((g["crk_m0"].shape[0], 10))
    vals[:, 0] = g["crk_m0"]
    vals[:, 1:4] = g["crk_m1"]
    m2 = g["crk_m2"]
    vals[:, 4], vals[:, 5], vals[:, 6] = m2[:, 0, 0], m2[:, 0, 1], m2[:, 0, 2]
    vals[:, 7], vals[:, 8], vals[:, 9] = m2[:, 1, 1], m2[:, 1, 2], m2[:, 2, 2]
    A, B, fb, *_ = oracle.crk_solve(vals, g["built_species"] == 1)
    np.testing.assert_array_equal(A, g["crk_A"])
    np.testing.assert_array_equal(B, g["crk_B"])
    np.testing.assert_array_equal(fb, g["crk_fallback"])
