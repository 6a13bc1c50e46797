"""GPU-vs-oracle parity at the benchmark configs (BASELINE.json configs[1..4]).

Each case runs the resident hb_force_step on the FULL workload bench.py
measures (same generator, same scales: bench.make_workload) and compares it
with the pinned oracle (tests/_parity.py):

* bit-exact over the whole set: the leaf permutation, the leaf count and the
  ordered list's entry count (hb/cmtree.py:125-196, 303-337);
* on sampled receiver leaves (every stride-th leaf plus every leaf of the most
  crowded bins; a receiver's outputs depend only on its own list entries, so
  the oracle's values there are exact): neighbour counts and CRK fallback flags
  bit-exact; density, CRK moments, A, B, gravity and hydro within
  tests/tolerances.py (hb/hydro.py:60-196, hb/kernels.py:143-278).

c3 (2x256^3, sigma_psi = 2 d: shell crossing, neighbour-count imbalance) is the
north star's parity target ("one full step on 2x256^3 matches the
reference").  c4 (2x512^3) is the benchmark's headline config and needs ~160
GB of device memory.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _workload(name):
    import bench
    p, cfg, meta = bench.make_workload(name)
    return p, cfg


@pytest.mark.parametrize("name,stride", [("c2", 16), ("c3", 128)])
def test_fullsize_step_vs_oracle(oracle, name, stride):
    from tests._parity import check_step
    p, cfg = _workload(name)
    st = check_step(oracle, p, cfg, stride, what=name)
    assert st["sampled_rows"] > 10000, st


def test_c4_step_vs_oracle(oracle):
    """The headline config (2x512^3) on one GPU: full-set leaf order and list
    size, ~1/4096 of the receivers against the oracle."""
    import torch
    free, total = torch.cuda.mem_get_info()
    if total < 170e9:
        pytest.skip("c4 needs ~160 GB of device memory")
    from tests._parity import check_step
    p, cfg = _workload("c4")
    st = check_step(oracle, p, cfg, 4096, what="c4")
    assert st["sampled_rows"] > 10000, st


def test_dark_matter_gravity_vs_oracle(oracle):
    """Single-species (configs[4]-like) gravity: a 512^3 dark-matter lattice,
    gravity pass only, sampled receivers against the oracle."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.resident import StepConfig
    from tests._parity import check_step
    npd = 512
    p = make_zeldovich_ic(npd, BoxGeometry(1.0), 0.05, species="dm")
    d = 1.0 / npd
    r_s, r_cut = d, 5 * d
    cfg = StepConfig(box=BoxGeometry(1.0), bin_width=max(4 * d / 2, r_cut * (1 + 1e-9)),
                     max_leaf_size=256, r_s=r_s, r_cut=r_cut,
                     softening=(1.0 / p.n ** (1 / 3)) / 50)
    st = check_step(oracle, p, cfg, 2048, what="dm512")
    assert st["sampled_rows"] > 10000, st


@pytest.mark.parametrize("npd", [24, 32])
def test_clustered_ic_step_vs_oracle(oracle, npd):
    """The reference's own clustered generator (hb/ic.py:137-169: 70% of the
    particles in 8 Gaussian clumps of sigma L/40, h = 1.3 d everywhere): bins
    far above the tiler's 2048 members, thousands of SPH neighbours per clump
    particle.  Every receiver leaf is compared (stride 1)."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_clustered_ic
    from paper_2510_03557_b200.resident import StepConfig
    from tests._parity import check_step
    box = BoxGeometry(1.0)
    p = make_clustered_ic(npd, box, seed=3)
    d = 1.0 / npd
    r_s, r_cut = d, 5 * d
    reach = max(r_cut, 2 * float(p.smoothing.max()))
    cfg = StepConfig(box=box, bin_width=max(2 * d, reach * (1 + 1e-9)), max_leaf_size=256,
                     r_s=r_s, r_cut=r_cut, softening=(1.0 / p.n ** (1 / 3)) / 50)
    check_step(oracle, p, cfg, 1 if npd <= 24 else 4, what=f"clustered{npd}")
