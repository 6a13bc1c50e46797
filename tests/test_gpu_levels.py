"""assign_timestep_levels on the device (csrc/hb_levels.cu) against the
reference's own output (tests/golden/levels.npz from hb/hydro.py:277-317):
row levels, leaf levels and the hierarchy depth bit for bit, flat and not,
and StiffStateError where the reference raises it."""
import numpy as np
import pytest

from tests.conftest import MeshView
from tests.test_gpu_parity import particle_set

pytestmark = pytest.mark.gpu


def _mesh(g):
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import ChainingMesh
    mv = MeshView(g, "mesh_")
    return ChainingMesh(box=BoxGeometry(1.0), bounds_lo=None, bounds_hi=None,
                        bin_count=mv.bin_count, bin_width=mv.bin_width,
                        periodic_axis=mv.periodic_axis, n_particles=int(mv.leaf_end[-1]),
                        leaf_start=mv.leaf_start, leaf_end=mv.leaf_end, leaf_lo=mv.leaf_lo,
                        leaf_hi=mv.leaf_hi, leaf_level=np.zeros_like(mv.leaf_level),
                        leaf_ghost_only=mv.leaf_ghost_only, leaf_bin=mv.leaf_bin,
                        _bin_ptr=mv._bin_ptr, _bin_ids=mv._bin_ids)


@pytest.mark.parametrize("flat", [False, True])
def test_levels_bitwise(golden, flat):
    from paper_2510_03557_b200.hydro import assign_timestep_levels
    g = golden("levels")
    p = particle_set(g, "in_")
    p.accel = np.array(g["in_accel"])
    mesh = _mesh(g)
    tag = "flat_" if flat else ""
    hier = assign_timestep_levels(p, mesh, float(g["dt_pm"]), float(g["cfl"]), 4,
                                  float(g["eps"]), 5 / 3, flat=flat)
    np.testing.assert_array_equal(p.timestep_level, g[tag + "level"])
    np.testing.assert_array_equal(mesh.leaf_level, g[tag + "leaf_level"])
    assert hier.max_level == int(g[tag + "max_level"])
    assert hier.n_fine == 1 << int(g[tag + "max_level"])


def test_levels_stiff_raises(golden):
    from paper_2510_03557_b200.errors import StiffStateError
    from paper_2510_03557_b200.hydro import assign_timestep_levels
    g = golden("levels")
    assert int(g["stiff_raises"]) == 1
    p = particle_set(g, "in_")
    p.accel = np.array(g["in_accel"])
    before = p.timestep_level.copy()
    with pytest.raises(StiffStateError, match="exceeds n_levels-1 = 3"):
        assign_timestep_levels(p, _mesh(g), 64 * float(g["dt_pm"]), float(g["cfl"]), 4,
                               float(g["eps"]), 5 / 3)
    np.testing.assert_array_equal(p.timestep_level, before)   # untouched, as the reference
