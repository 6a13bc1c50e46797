"""Debug: per-kernel momentum-quanta residual of deterministic mirror evals."""
import numpy as np, sys
sys.path.insert(0, '.')
from tests.conftest import MeshView
from tests.test_gpu_subcycle import _inputs
from paper_2510_03557_b200.kernels import gravity_kernel, hydro_force_kernel
from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
from paper_2510_03557_b200.cmtree import assemble_interaction_lists, InteractionList
from paper_2510_03557_b200.stepper import unordered_due_pairs
g = dict(np.load('tests/golden/subcycle.npz'))
p, mesh, box = _inputs(g)
il = assemble_interaction_lists(mesh, float(g['reach']), 0)
a, b, sh, lev = unordered_due_pairs(il, mesh)
from paper_2510_03557_b200.hydro import compute_density, refresh_eos_columns
st = p.state_matrix(5/3)
compute_density(p, mesh, st, il, mode=EvalMode.DETERMINISTIC)
refresh_eos_columns(st, p, 5/3)
same = (a == b) & np.all(sh == 0, axis=1)
for name, k in (('grav', gravity_kernel(float(g['r_s']), float(g['r_cut']), float(g['eps']))),
                ('hydro', hydro_force_kernel(2 * p.smoothing.max(), 1.0, 2.0))):
    for sel_name, sel in (('all', np.ones_like(same)), ('same', same), ('cross', ~same)):
        sub = InteractionList(a[sel], b[sel], il.reach, 0, sh[sel])
        r = eval_interaction_list(k, sub, st, mesh, mode=EvalMode.DETERMINISTIC, mirror=True,
                                  pshift=p.image_shift)
        print(name, sel_name, int(sel.sum()), r.int_acc[:, 0:3].sum(axis=0))
