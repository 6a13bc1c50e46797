"""Short-range side of the Gaussian force split (hb/gravity.py:37-55, 227-240).

S(x) = erfc(x) + 2x/sqrt(pi) e^{-x^2}, x = r / r_s, Plummer softening, cut at
r_cut = 5 r_s.  The long-range PM solver is out of scope."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .box import BoxGeometry
from .errors import HydroboxError
from .kernels import PairKernel, gravity_kernel, gravity_potential_kernel


@dataclass(frozen=True)
class ForceSplit:
    r_s: float
    r_cut: float

    @staticmethod
    def for_grid(box: BoxGeometry, grid_n: int, r_s: float | None = None,
                 r_cut_factor: float = 5.0) -> "ForceSplit":
        spacing = box.side_length / grid_n
        rs = 2.0 * spacing if r_s is None else r_s
        return ForceSplit(r_s=rs, r_cut=r_cut_factor * rs)

    def short_fraction(self, r) -> np.ndarray:
        x = np.asarray(r, dtype=np.float64) / self.r_s
        erfc = np.vectorize(math.erfc, otypes=[np.float64])
        return erfc(x) + (2.0 / math.sqrt(math.pi)) * x * np.exp(-x * x)


def short_range_gravity_kernel(split: ForceSplit, softening: float) -> PairKernel:
    """Momentum-rate channels m_i a_i of the short-range force; refuses a cutoff
    whose tail S(r_cut) >= 1e-5 (hb/gravity.py:227-235)."""
    if float(split.short_fraction(split.r_cut)) >= 1e-5:
        raise HydroboxError("r_cut too small: short-range tail exceeds 1e-5")
    return gravity_kernel(split.r_s, split.r_cut, softening)


def short_range_potential_kernel(split: ForceSplit, softening: float) -> PairKernel:
    return gravity_potential_kernel(split.r_s, split.r_cut, softening)
