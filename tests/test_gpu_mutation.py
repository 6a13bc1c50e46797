"""Negative controls for the parity checker (tests/_parity.py): a step with a
seeded defect must FAIL the oracle comparison.  Each mutation is applied to the
GPU side only -- the oracle always sees the true configuration -- so a checker
that passed these would be blind to that class of bug:

* r_cut shrunk by 0.1% on the GPU: the lost sources sit where S(r/r_s) < 1e-5,
  invisible in the normalised force error; the list size or the exact in-r_cut
  counts catch it;
* the artificial viscosity term dropped (alpha = beta = 0, hb/kernels.py:240-250);
* one gas particle's smoothing length lowered by 1% (neighbour counts, density).
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _c1():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.resident import StepConfig
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(32, box, 1.0)
    d = 1.0 / 32
    reach = max(5 * d, 2 * float(p.smoothing.max()))
    cfg = StepConfig(box=box, bin_width=reach * (1 + 1e-9), max_leaf_size=256, r_s=d,
                     r_cut=5 * d, softening=(1.0 / p.n ** (1 / 3)) / 50)
    return p, cfg


def test_unmutated_step_passes(oracle):
    from tests._parity import check_step
    p, cfg = _c1()
    check_step(oracle, p, cfg, 4, what="control")


@pytest.mark.parametrize("mutation,match", [("r_cut", "r_cut"), ("viscosity", "hydro"),
                                            ("smoothing", "neighbour counts|density")])
def test_mutated_step_fails(oracle, mutation, match):
    from paper_2510_03557_b200.resident import ResidentRank
    from tests._parity import check_step
    p, cfg = _c1()
    q = p.copy()
    gcfg = cfg
    if mutation == "r_cut":
        gcfg = dataclasses.replace(cfg, r_cut=cfg.r_cut * 0.999)
    elif mutation == "viscosity":
        gcfg = dataclasses.replace(cfg, visc_alpha=0.0, visc_beta=0.0)
    else:
        g = np.nonzero(q.species == 1)[0]
        q.smoothing[g[len(g) // 2]] *= 0.99   # below h_max: the list is unchanged
    rank = ResidentRank(q, gcfg)
    with pytest.raises(AssertionError, match=match):
        check_step(oracle, p, cfg, 1, what=f"mutation {mutation}", rank=rank)
