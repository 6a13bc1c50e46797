"""Separation-of-scales gravity (hb/gravity.py): the short-range side of the
Gaussian split and the spectral particle-mesh long range.

Short range: S(x) = erfc(x) + 2x/sqrt(pi) e^{-x^2}, x = r / r_s, Plummer
softening, cut at r_cut = 5 r_s (the force path, hb_pairs.cu).
Long range, on the device: CIC deposit (hb_pm_deposit),
cuFFT R2C, the alias-optimal influence function D(k) (evaluated on the GPU,
cached per grid), phi_k = -4 pi G rho_k D(k) and the three -i k phi_k force
spectra (hb_pm_spectral), cuFFT C2R, CIC interpolation (hb_pm_interp)."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

import ctypes as C

from . import _native as N
from .box import BoxGeometry
from .errors import HydroboxError
from .kernels import PairKernel, gravity_kernel, gravity_potential_kernel
from .particles import ParticleSet

G_NEWTON = 1.0  # code units (hb/gravity.py:24)


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


# ------------------------------------------------------------------ long range
@dataclass
class MeshField:
    """Samples on the PM grid, values at cell centres (hb/gravity.py:27-33).
    ``values`` is a numpy array in the compat API, a CUDA tensor on the device path."""

    grid_n: int
    spacing: float
    values: object


def _axes(grid_n: int, box: BoxGeometry):
    """The reference's k axes, bit for bit (2 pi * np.fft.(r)fftfreq)."""
    L, n = box.side_length, grid_n
    return (2.0 * math.pi * np.fft.fftfreq(n, d=L / n),
            2.0 * math.pi * np.fft.rfftfreq(n, d=L / n))


_INFLUENCE: dict = {}


def optimal_influence_device(grid_n: int, box: BoxGeometry, r_s: float):
    """Alias-optimal scalar influence function of the CIC deposit -> ik ->
    CIC interpolate pipeline for the Gaussian target force (Hockney-Eastwood;
    hb/gravity.py:87-140), summed over 5^3 alias images on the device.
    (n, n, n/2+1) float64 tensor, cached per (grid, box, r_s)."""
    torch = N.torch_cuda()
    dev = torch.cuda.current_device()
    key = (dev, grid_n, round(box.side_length, 12), round(r_s, 12))
    if key in _INFLUENCE:
        return _INFLUENCE[key]
    L, n = box.side_length, grid_n
    kg = 2.0 * math.pi * n / L
    k1, k3 = (torch.from_numpy(a).cuda() for a in _axes(n, box))
    kx, ky, kz = k1[:, None, None], k1[None, :, None], k3[None, None, :]

    def w1sq(k):
        return torch.sinc(k * (L / n) / 2.0 / math.pi) ** 4

    imgs = range(-2, 3)
    num = torch.zeros((n, n, n // 2 + 1), dtype=torch.float64, device="cuda")
    for mx in imgs:
        kmx = kx + mx * kg
        wx = w1sq(kmx)
        for my in imgs:
            kmy = ky + my * kg
            wxy = wx * w1sq(kmy)
            for mz in imgs:
                kmz = kz + mz * kg
                km2 = kmx ** 2 + kmy ** 2 + kmz ** 2
                km2 = torch.where(km2 == 0, torch.ones_like(km2), km2)
                g = torch.exp(-km2 * (r_s * r_s) / 4.0) / km2
                num += (kx * kmx + ky * kmy + kz * kmz) * g * (wxy * w1sq(kmz))

    def axis_sum(k):
        return sum(w1sq(k + m * kg) for m in imgs)
    denom = (axis_sum(kx) * axis_sum(ky) * axis_sum(kz)) ** 2
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    d = num / (torch.where(k2 == 0, torch.ones_like(k2), k2) * denom)
    d[0, 0, 0] = 0.0
    _INFLUENCE[key] = d
    return d


def naive_influence_device(grid_n: int, box: BoxGeometry, r_s: float):
    """exp(-k^2 r_s^2 / 4) / (k^2 W_cic^2) (hb/gravity.py:69-85)."""
    torch = N.torch_cuda()
    n = grid_n
    k1, k3 = (torch.from_numpy(a).cuda() for a in _axes(n, box))
    kx, ky, kz = k1[:, None, None], k1[None, :, None], k3[None, None, :]
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    k2[0, 0, 0] = 1.0
    m1 = torch.from_numpy(np.fft.fftfreq(n) * n).cuda()
    m3 = torch.from_numpy(np.fft.rfftfreq(n) * n).cuda()
    wx = torch.sinc(m1 / n)[:, None, None] ** 2
    wy = torch.sinc(m1 / n)[None, :, None] ** 2
    wz = torch.sinc(m3 / n)[None, None, :] ** 2
    return torch.exp(-k2 * (r_s * r_s) / 4.0) / (k2 * (wx * wy * wz) ** 2)


def deposit_cic_device(pos_d, mass_d, grid_n: int, box: BoxGeometry):
    """(n, n, n) float64 mass density on the device (hb/gravity.py:69-82)."""
    torch = N.torch_cuda()
    spacing = box.side_length / grid_n
    rho = torch.empty((grid_n, grid_n, grid_n), dtype=torch.float64, device="cuda")
    err = N.HbError()
    N.check(N.lib().hb_pm_deposit(int(pos_d.shape[0]), N.ptr(pos_d), N.ptr(mass_d), grid_n,
                                  spacing, spacing ** 3, N.ptr(rho), N.stream_ptr(),
                                  C.byref(err)), err)
    return rho


def solve_long_range_device(rho_d, split: "ForceSplit", box: BoxGeometry,
                            want_potential: bool = False, influence: str = "optimal"):
    """Filtered spectral Poisson solve on the device (hb/gravity.py:143-216):
    ([fx, fy, fz] grids, potential grid or None)."""
    torch = N.torch_cuda()
    n = int(rho_d.shape[0])
    spacing = box.side_length / n
    if split.r_s < spacing:
        raise HydroboxError(f"split scale {split.r_s:.4g} is below one grid "
                            f"spacing {spacing:.4g}")
    if influence == "optimal":
        d_k = optimal_influence_device(n, box, split.r_s)
    elif influence == "naive":
        d_k = naive_influence_device(n, box, split.r_s)
    else:
        raise HydroboxError(f"unknown influence '{influence}'")
    # cuFFT's R2C result comes back with the half axis outermost in memory:
    # the spectral kernel works on row-major (n, n, n/2+1)
    rho_k = torch.fft.rfftn(rho_d).contiguous()
    spec = [torch.empty(rho_k.shape, dtype=rho_k.dtype, device="cuda")
            for _ in range(4 if want_potential else 3)]
    err = N.HbError()
    N.check(N.lib().hb_pm_spectral(n, float(box.side_length), 4.0 * math.pi * G_NEWTON,
                                   N.ptr(rho_k), N.ptr(d_k.contiguous()), N.ptr(spec[0]),
                                   N.ptr(spec[1]), N.ptr(spec[2]),
                                   N.ptr(spec[3]) if want_potential else None,
                                   N.stream_ptr(), C.byref(err)), err)
    grids = [torch.fft.irfftn(f, s=(n, n, n)) for f in spec]
    return grids[:3], (grids[3] if want_potential else None)


def interpolate_device(grids, pos_d, spacing: float):
    """CIC gather of 1..3 grids at the positions: (np, len(grids)) float64."""
    torch = N.torch_cuda()
    npt = int(pos_d.shape[0])
    out = torch.empty((npt, len(grids)), dtype=torch.float64, device="cuda")
    g = [x.contiguous() for x in grids] + [None] * (3 - len(grids))
    err = N.HbError()
    N.check(N.lib().hb_pm_interp(npt, N.ptr(pos_d), len(grids), N.ptr(g[0]), N.ptr(g[1]),
                                 N.ptr(g[2]), int(grids[0].shape[0]), spacing, N.ptr(out),
                                 N.stream_ptr(), C.byref(err)), err)
    return out


class LongRangeSolver:
    """Device-resident PM long range for one grid: deposit -> solve -> gather,
    reusing the cached influence function; positions / masses stay on the GPU."""

    def __init__(self, grid_n: int, split: "ForceSplit", box: BoxGeometry,
                 influence: str = "optimal"):
        self.grid_n, self.split, self.box, self.influence = grid_n, split, box, influence
        self.spacing = box.side_length / grid_n

    def accelerations(self, pos_d, mass_d, want_potential: bool = False):
        rho = deposit_cic_device(pos_d, mass_d, self.grid_n, self.box)
        fields, pot = solve_long_range_device(rho, self.split, self.box, want_potential,
                                              self.influence)
        acc = interpolate_device(fields, pos_d, self.spacing)
        if not want_potential:
            return acc, None
        return acc, interpolate_device([pot], pos_d, self.spacing)[:, 0]


# compat API: the reference's host-array signatures (hb/gravity.py:69-245)
def deposit_cic(particles: ParticleSet, grid_n: int, box: BoxGeometry) -> MeshField:
    rho = deposit_cic_device(N.dev(np.ascontiguousarray(particles.pos)),
                             N.dev(np.ascontiguousarray(particles.mass)), grid_n, box)
    return MeshField(grid_n=grid_n, spacing=box.side_length / grid_n, values=rho.cpu().numpy())


def solve_long_range(density: MeshField, split: "ForceSplit", box: BoxGeometry,
                     want_potential: bool = False, influence: str = "optimal"):
    fields, pot = solve_long_range_device(N.dev(np.ascontiguousarray(density.values)), split,
                                          box, want_potential, influence)
    out = [MeshField(grid_n=density.grid_n, spacing=density.spacing, values=f.cpu().numpy())
           for f in fields]
    if want_potential:
        return out, MeshField(grid_n=density.grid_n, spacing=density.spacing,
                              values=pot.cpu().numpy())
    return out


def interpolate_force(fields: list, particles: ParticleSet) -> np.ndarray:
    grids = [N.dev(np.ascontiguousarray(f.values)) for f in fields]
    out = interpolate_device(grids, N.dev(np.ascontiguousarray(particles.pos)),
                             fields[0].spacing).cpu().numpy()
    res = np.zeros((particles.n, 3))  # the reference returns (n, 3) for any field count
    res[:, :out.shape[1]] = out
    return res


def interpolate_scalar(field: MeshField, particles: ParticleSet) -> np.ndarray:
    return interpolate_force([field], particles)[:, 0]


def long_range_potential_energy(pot: MeshField, particles: ParticleSet) -> float:
    """1/2 sum over owned rows of m_i phi(r_i) (hb/gravity.py:240-245)."""
    phi = interpolate_scalar(pot, particles)
    own = particles.owned_mask()
    return 0.5 * float(np.sum(particles.mass[own] * phi[own]))
