"""Pair-kernel descriptors, id-for-id with the reference registry
(hb/kernels.py:33-61, 436-602).  The arithmetic itself lives in
csrc/hb_pairs.cuh; these objects carry the ids, channel layout, reach,
params, mirror rules, determinism scales and FLOP-proxy costs that the C ABI
(HbEvalArgs) takes."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KID_COUNTING = 0
KID_GRAVITY = 1
KID_GRAV_POT = 2
KID_DENSITY = 3
KID_CRK_MOMENTS = 4
KID_HYDRO_FORCE = 5
KID_NEIGHBOR_COUNT = 6
KID_STUB_ZERO = 7
KID_CRK_INTERP = 8
KID_CRK_GRAD1 = 9   # CRK gradient moments (north star; not in the reference)
KID_CRK_GRAD2 = 10

GAS = 1.0

CNT_F_EVALS, CNT_G_EVALS, CNT_ROT_ITERS, CNT_PAIRS_SCHED, CNT_PAIRS_IN = 0, 1, 2, 3, 4
CNT_ERR_KIND, CNT_ERR_A, CNT_ERR_B, N_COUNTERS = 5, 6, 7, 8
ERR_NONE, ERR_NONFINITE, ERR_OVERFLOW = 0, 1, 2

QGUARD = 2.0 ** 56
ACC_GUARD = np.int64(2) ** 62


@dataclass(frozen=True)
class OpCost:
    """FLOP proxy of one pair evaluation (FMA = 2 ops), hb/kernels.py:436-446."""

    adds: int = 0
    muls: int = 0
    fmas: int = 0
    special: int = 0

    def total(self) -> int:
        return self.adds + self.muls + 2 * self.fmas + self.special


class Symmetry:
    SYMMETRIC = "symmetric"
    ANTISYMMETRIC = "antisymmetric"
    NONE = "none"


@dataclass(frozen=True)
class PairKernel:
    name: str
    kid: int
    n_channels: int
    channel_names: tuple
    load_i: tuple
    load_j: tuple
    symmetry: str
    include_self: bool
    reach: float
    params: np.ndarray
    channel_signs: np.ndarray
    scale_bits: tuple
    op_cost: OpCost
    mirrorable: bool = True
    n_aux: int = 0
    mirror_swap: np.ndarray | None = None

    @property
    def scales(self) -> np.ndarray:
        return np.array([2.0 ** b for b in self.scale_bits])

    @property
    def mirror_map(self) -> np.ndarray:
        if self.mirror_swap is not None:
            return self.mirror_swap
        return np.arange(self.n_channels, dtype=np.int64)


def _k(name, kid, names, li, lj, sym, self_, reach, params, signs, bits, cost, **kw):
    return PairKernel(name=name, kid=kid, n_channels=len(names), channel_names=names,
                      load_i=li, load_j=lj, symmetry=sym, include_self=self_, reach=reach,
                      params=np.asarray(params, dtype=np.float64),
                      channel_signs=np.asarray(signs, dtype=np.int64), scale_bits=bits,
                      op_cost=cost, **kw)


def counting_kernel(reach: float) -> PairKernel:
    return _k("counting", KID_COUNTING, ("count",), (), (), Symmetry.SYMMETRIC, False, reach,
              [0.0], [1], (40,), OpCost(adds=1))


def stub_zero_kernel(reach: float) -> PairKernel:
    return _k("stub_zero", KID_STUB_ZERO, ("zero",), (), (), Symmetry.SYMMETRIC, False, reach,
              [0.0], [1], (40,), OpCost(adds=1))


def gravity_kernel(split_scale: float, r_cut: float, softening: float) -> PairKernel:
    """Short-range complement of the Gaussian split (hb/kernels.py:513-523)."""
    return _k("gravity_short", KID_GRAVITY, ("fx", "fy", "fz"), ("mass",), ("mass",),
              Symmetry.ANTISYMMETRIC, False, r_cut, [split_scale, softening * softening],
              [-1, -1, -1], (44, 44, 44), OpCost(adds=8, muls=12, fmas=3, special=3))


def gravity_potential_kernel(split_scale: float, r_cut: float, softening: float) -> PairKernel:
    return _k("gravity_pot", KID_GRAV_POT, ("pe",), ("mass",), ("mass",), Symmetry.SYMMETRIC,
              False, r_cut, [split_scale, softening * softening], [1], (44,),
              OpCost(adds=5, muls=6, special=2))


def density_kernel(reach: float) -> PairKernel:
    return _k("density", KID_DENSITY, ("rho",), ("smoothing",), ("mass",), Symmetry.NONE, True,
              reach, [0.0], [1], (50,), OpCost(adds=6, muls=9, special=1), mirrorable=False)


def neighbor_count_kernel(reach: float) -> PairKernel:
    return _k("neighbor_count", KID_NEIGHBOR_COUNT, ("count",), ("smoothing",), (),
              Symmetry.NONE, True, reach, [0.0], [1], (40,), OpCost(adds=4, muls=3),
              mirrorable=False)


def crk_moments_kernel(reach: float) -> PairKernel:
    return _k("crk_moments", KID_CRK_MOMENTS,
              ("m0", "m1x", "m1y", "m1z", "m2xx", "m2xy", "m2xz", "m2yy", "m2yz", "m2zz"),
              ("smoothing",), ("mass", "density"), Symmetry.NONE, True, reach, [0.0],
              np.ones(10, dtype=np.int64), (52,) * 10, OpCost(adds=10, muls=18, special=1),
              mirrorable=False)


def crk_gradient_kernels(reach: float) -> tuple:
    """Gradient moments for gradA / gradB (the north star's CRK gradients; the
    reference has none): with G = V_j (dW/dr)/r at h_i and dr = x_i - x_j,
    GRAD1 = [sum G dr (3), sum G dr dr (xx xy xz yy yz zz)],
    GRAD2 = sum G dr dr dr (xxx xxy xxz xyy xyz xzz yyy yyz yzz zzz)."""
    g1 = _k("crk_grad1", KID_CRK_GRAD1,
            ("gx", "gy", "gz", "gxx", "gxy", "gxz", "gyy", "gyz", "gzz"),
            ("smoothing",), ("mass", "density"), Symmetry.NONE, True, reach, [0.0],
            np.ones(9, dtype=np.int64), (48,) * 9, OpCost(adds=9, muls=14, special=1),
            mirrorable=False)
    g2 = _k("crk_grad2", KID_CRK_GRAD2,
            ("gxxx", "gxxy", "gxxz", "gxyy", "gxyz", "gxzz", "gyyy", "gyyz", "gyzz", "gzzz"),
            ("smoothing",), ("mass", "density"), Symmetry.NONE, True, reach, [0.0],
            np.ones(10, dtype=np.int64), (44,) * 10, OpCost(adds=10, muls=18, special=1),
            mirrorable=False)
    return g1, g2


def crk_interp_kernel(reach: float) -> PairKernel:
    """Corrected interpolation; aux = [F_j, A, Bx, By, Bz] (hb/kernels.py:571-580)."""
    return _k("crk_interp", KID_CRK_INTERP, ("fhat",), ("smoothing",), ("mass", "density"),
              Symmetry.NONE, True, reach, [0.0], [1], (48,), OpCost(adds=8, muls=12, special=1),
              mirrorable=False, n_aux=5)


def hydro_force_kernel(reach: float, visc_alpha: float = 1.0, visc_beta: float = 2.0) -> PairKernel:
    """SPH momentum + energy rate with Monaghan viscosity (hb/kernels.py:583-602)."""
    return _k("hydro_force", KID_HYDRO_FORCE, ("fx", "fy", "fz", "edot_i", "edot_j"),
              ("mass", "pressure", "density"), ("mass", "pressure", "density"), Symmetry.NONE,
              False, reach, [visc_alpha, visc_beta], [-1, -1, -1, 1, 1], (44,) * 5,
              OpCost(adds=18, muls=26, fmas=6, special=1),
              mirror_swap=np.array([0, 1, 2, 4, 3], dtype=np.int64))
