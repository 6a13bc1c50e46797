import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
        return cache[name]
    return load


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


class MeshView:
    """Minimal mesh object from golden arrays (fields the engine reads)."""

    def __init__(self, g, prefix, L=1.0):
        from paper_2510_03557_b200.box import BoxGeometry
        self.box = BoxGeometry(L)
        self.leaf_start = g[prefix + "leaf_start"]
        self.leaf_end = g[prefix + "leaf_end"]
        self.leaf_lo = g[prefix + "leaf_lo"]
        self.leaf_hi = g[prefix + "leaf_hi"]
        self.leaf_level = g[prefix + "leaf_level"]
        self.leaf_ghost_only = g[prefix + "leaf_ghost_only"]
        self.leaf_bin = g[prefix + "leaf_bin"]
        self.bin_count = g[prefix + "bin_count"]
        self.bin_width = g[prefix + "bin_width"]
        self.periodic_axis = g[prefix + "periodic"]
        self._bin_ptr = g[prefix + "bin_ptr"]
        self._bin_ids = g[prefix + "bin_ids"]
        self.n_particles = int(self.leaf_end[-1]) if self.leaf_end.size else 0

    @property
    def n_leaves(self):
        return self.leaf_start.shape[0]
