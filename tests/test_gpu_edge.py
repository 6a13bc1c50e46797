"""GPU edge cases the reference handles: empty particle sets, an empty
interaction list, a lone particle (self term only), a two-particle pair."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(box, bw=0.25):
    from paper_2510_03557_b200.resident import StepConfig
    return StepConfig(box=box, bin_width=bw, max_leaf_size=256, r_s=0.02, r_cut=0.1,
                      softening=1e-3)


def _lone(n_gas=1):
    from paper_2510_03557_b200.particles import ParticleSet
    p = ParticleSet(n_gas)
    p.pos[:] = np.array([[0.31, 0.52, 0.73]])[:n_gas] if n_gas == 1 else \
        np.array([[0.31, 0.52, 0.73], [0.33, 0.52, 0.73]])
    p.mass[:] = 1e-3
    p.species[:] = 1
    p.smoothing[:] = 0.02
    p.internal_energy[:] = 1e-4
    p.global_id = np.arange(n_gas, dtype=np.int64)
    return p


def test_empty_set():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.particles import ParticleSet
    from paper_2510_03557_b200.resident import force_step
    box = BoxGeometry(1.0)
    p = ParticleSet(0)
    mesh = build_mesh_and_leaves(p, box, 0.25, 64)
    assert mesh.n_leaves == 0
    il = assemble_interaction_lists(mesh, 0.2, 0)
    assert len(il) == 0
    out = force_step(ParticleSet(0), _cfg(box))
    assert out["grav"].shape[0] == 0 and out["ncount"].shape[0] == 0


def test_empty_list_evaluates_to_zeros():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import InteractionList, build_mesh_and_leaves
    from paper_2510_03557_b200.kernels import density_kernel
    from paper_2510_03557_b200.lane import eval_interaction_list
    box = BoxGeometry(1.0)
    p = _lone()
    mesh = build_mesh_and_leaves(p, box, 0.25, 64)
    il = InteractionList(np.zeros(0, np.int64), np.zeros(0, np.int64), 0.2, 0)
    res = eval_interaction_list(density_kernel(0.04), il, p.state_matrix(5 / 3), mesh)
    assert res.values.shape == (1, 1) and not res.values.any()


@pytest.mark.parametrize("n_gas", [1, 2])
def test_lone_and_pair(n_gas):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.resident import force_step
    box = BoxGeometry(1.0)
    p = _lone(n_gas)
    out = force_step(p, _cfg(box))
    sig = 1.0 / math.pi
    h = 0.02
    if n_gas == 1:
        np.testing.assert_array_equal(out["ncount"], [1.0])
        np.testing.assert_allclose(p.density, [1e-3 * sig / h ** 3], rtol=1e-6)
        np.testing.assert_array_equal(out["grav"], np.zeros((1, 3)))
    else:
        q = 0.02 / h        # separation 0.02 = h: W(1) = 1/4
        np.testing.assert_array_equal(out["ncount"], [2.0, 2.0])
        np.testing.assert_allclose(p.density, [1e-3 * sig / h ** 3 * (1 + 0.25)] * 2, rtol=1e-6)
        g = out["grav"]
        np.testing.assert_allclose(g[0], -g[1], rtol=1e-6)   # equal and opposite
        assert abs(g[0, 0]) > 0 and q == 1.0
