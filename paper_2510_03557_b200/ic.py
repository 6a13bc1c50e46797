"""Deterministic initial conditions: the reference's two-species lattice and
clustered sets (hb/ic.py:27-62, 137-169) and the Zel'dovich-displaced lattice
the benchmark configs name (not in the reference -- SPEC.md:108 lists it as a
non-goal -- so it is generated here and fed identically to every arm)."""
from __future__ import annotations

import numpy as np

from .box import BoxGeometry, wrap_position
from .errors import ConfigError
from .particles import ParticleSet, Species

ZELDOVICH_SEED = 2510035570


def _lattice(n: int, spacing: float, origin: float) -> np.ndarray:
    axis = origin + spacing * np.arange(n)
    gx, gy, gz = np.meshgrid(axis, axis, axis, indexing="ij")
    return np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])


def _two_species(n_per_dim: int, box: BoxGeometry, dm_pos, gas_pos,
                 gas_internal_energy: float) -> ParticleSet:
    n_site = n_per_dim ** 3
    spacing = box.side_length / n_per_dim
    p = ParticleSet(2 * n_site)
    p.pos = wrap_position(np.vstack([dm_pos, gas_pos]), box)
    p.mass[:] = box.volume / (2 * n_site)
    p.species[:n_site] = Species.DARK_MATTER
    p.species[n_site:] = Species.GAS
    p.smoothing[n_site:] = 1.3 * spacing
    p.internal_energy[n_site:] = gas_internal_energy
    p.global_id = np.arange(2 * n_site, dtype=np.int64)
    return p


def make_lattice_ic(n_per_dim: int, box: BoxGeometry, perturbation_amplitude: float = 0.0,
                    seed: int = 0, gas_internal_energy: float = 1e-4) -> ParticleSet:
    """DM lattice at 0.25 d plus gas at 0.75 d, uniform jitter (hb/ic.py:27-62)."""
    if n_per_dim < 2:
        raise ConfigError("n_per_dim must be >= 2")
    spacing = box.side_length / n_per_dim
    if perturbation_amplitude >= 0.5 * spacing:
        raise ConfigError("perturbation amplitude must stay below half the lattice spacing")
    dm = _lattice(n_per_dim, spacing, 0.25 * spacing)
    gas = _lattice(n_per_dim, spacing, 0.75 * spacing)
    rng = np.random.default_rng(seed)
    if perturbation_amplitude > 0:
        dm = dm + rng.uniform(-perturbation_amplitude, perturbation_amplitude, dm.shape)
        gas = gas + rng.uniform(-perturbation_amplitude, perturbation_amplitude, gas.shape)
    return _two_species(n_per_dim, box, dm, gas, gas_internal_energy)


def zeldovich_displacement(n_per_dim: int, box: BoxGeometry, sigma_psi: float,
                           seed: int = ZELDOVICH_SEED) -> np.ndarray:
    """Displacement field psi (n^3, 3) on the lattice: Gaussian delta(k) with
    P(k) ~ k^-2 exp(-(k d)^2), psi(k) = i k delta(k) / k^2 (k = 0 removed),
    rescaled to rms |psi| = sigma_psi.  float64, deterministic in `seed`."""
    n = n_per_dim
    L = box.side_length
    d = L / n
    rng = np.random.default_rng(seed)
    white = rng.standard_normal((n, n, n))
    dk = np.fft.rfftn(white)
    k1 = 2 * np.pi * np.fft.fftfreq(n, d=d)
    kz = 2 * np.pi * np.fft.rfftfreq(n, d=d)
    KX, KY, KZ = np.meshgrid(k1, k1, kz, indexing="ij")
    k2 = KX ** 2 + KY ** 2 + KZ ** 2
    k2[0, 0, 0] = 1.0
    amp = np.sqrt(np.exp(-k2 * d * d) / k2)   # sqrt(P(k)), P ~ k^-2 exp(-(kd)^2)
    amp[0, 0, 0] = 0.0
    dk *= amp
    psi = np.empty((n ** 3, 3))
    for comp, K in enumerate((KX, KY, KZ)):
        psi[:, comp] = np.fft.irfftn(1j * K / k2 * dk, s=(n, n, n), axes=(0, 1, 2)).ravel()
    rms = np.sqrt(np.mean(np.sum(psi ** 2, axis=1)))
    if rms > 0:
        psi *= sigma_psi / rms
    return psi


def make_zeldovich_ic(n_per_dim: int, box: BoxGeometry, sigma_psi_cells: float,
                      seed: int = ZELDOVICH_SEED, velocity_factor: float = 0.1,
                      gas_internal_energy: float = 1e-4, species: str = "both",
                      select=None) -> ParticleSet:
    """Two interleaved lattices displaced by the same psi.

    sigma_psi_cells: rms displacement in lattice spacings (0.05 ~ z=10,
    2 ~ z=0).  species='dm' gives the single-species gravity-only set.
    select: optional callable(pos (m,3)) -> bool mask; only the selected
    particles are materialised (e.g. one rank's domain), with the values and
    global ids they have in the full set, in the same order."""
    spacing = box.side_length / n_per_dim
    psi = zeldovich_displacement(n_per_dim, box, sigma_psi_cells * spacing, seed)
    if select is not None:
        return _zeldovich_subset(n_per_dim, box, psi, velocity_factor, gas_internal_energy,
                                 species, select)
    vel = velocity_factor * psi
    if species == "dm":
        n3 = n_per_dim ** 3
        p = ParticleSet(n3)
        p.pos = wrap_position(_lattice(n_per_dim, spacing, 0.5 * spacing) + psi, box)
        p.vel = vel.copy()
        p.mass[:] = box.volume / n3
        p.species[:] = Species.DARK_MATTER
        p.global_id = np.arange(n3, dtype=np.int64)
        return p
    dm = _lattice(n_per_dim, spacing, 0.25 * spacing) + psi
    gas = _lattice(n_per_dim, spacing, 0.75 * spacing) + psi
    p = _two_species(n_per_dim, box, dm, gas, gas_internal_energy)
    p.vel = np.vstack([vel, vel])
    return p


def _zeldovich_subset(n_per_dim, box, psi, velocity_factor, gas_internal_energy, species,
                      select) -> ParticleSet:
    """Selected rows of make_zeldovich_ic's set, built species by species so
    the full particle arrays never exist at once."""
    n3 = n_per_dim ** 3
    spacing = box.side_length / n_per_dim
    lattices = ([(Species.DARK_MATTER, 0.5, 0)] if species == "dm"
                else [(Species.DARK_MATTER, 0.25, 0), (Species.GAS, 0.75, n3)])
    n_all = n3 * len(lattices)
    parts = []
    for sp, origin, id0 in lattices:
        pos = wrap_position(_lattice(n_per_dim, spacing, origin * spacing) + psi, box)
        idx = np.nonzero(select(pos))[0]
        parts.append((sp, idx, pos[idx], id0))
        del pos
    p = ParticleSet(sum(len(x[1]) for x in parts))
    o = 0
    for sp, idx, pos, id0 in parts:
        k = len(idx)
        sl = slice(o, o + k)
        p.pos[sl] = pos
        p.vel[sl] = velocity_factor * psi[idx]
        p.mass[sl] = box.volume / n_all
        p.species[sl] = sp
        if sp == Species.GAS:
            p.smoothing[sl] = 1.3 * spacing
            p.internal_energy[sl] = gas_internal_energy
        p.global_id[sl] = idx + id0
        o += k
    return p


def make_zeldovich_ic_device(n_per_dim: int, box: BoxGeometry, sigma_psi_cells: float,
                             select, seed: int = ZELDOVICH_SEED, velocity_factor: float = 0.1,
                             gas_internal_energy: float = 1e-4,
                             species: str = "both") -> ParticleSet:
    """make_zeldovich_ic(select=...) with the displacement field built on the
    GPU (cuFFT), for sizes whose numpy field does not fit the host per rank
    (1024^3: ~60 GB).  The white noise is numpy's (same seed, same values); the
    FFTs are cuFFT's, so positions agree with the numpy set to rounding, not
    bitwise.  select: callable(pos torch (m,3) float64 CUDA) -> bool mask."""
    import torch
    n = n_per_dim
    L = box.side_length
    d = L / n
    dev = torch.device("cuda")
    white = torch.from_numpy(np.random.default_rng(seed).standard_normal((n, n, n))).to(dev)
    dk = torch.fft.rfftn(white)
    del white
    k1 = 2 * np.pi * torch.fft.fftfreq(n, d=d, dtype=torch.float64, device=dev)
    kz = 2 * np.pi * torch.fft.rfftfreq(n, d=d, dtype=torch.float64, device=dev)
    k2 = k1[:, None, None] ** 2 + k1[None, :, None] ** 2 + kz[None, None, :] ** 2
    k2[0, 0, 0] = 1.0
    amp = torch.sqrt(torch.exp(-k2 * d * d) / k2)
    amp[0, 0, 0] = 0.0
    dk *= amp
    del amp
    psi = torch.empty((3, n, n, n), dtype=torch.float64, device=dev)
    for comp, K in enumerate((k1[:, None, None], k1[None, :, None], kz[None, None, :])):
        psi[comp] = torch.fft.irfftn(1j * K / k2 * dk, s=(n, n, n))
    del dk, k2
    rms = torch.sqrt(torch.mean(torch.sum(psi ** 2, dim=0)))
    if float(rms) > 0:
        psi *= sigma_psi_cells * d / rms
    psi = psi.reshape(3, -1)
    lattices = ([(Species.DARK_MATTER, 0.5, 0)] if species == "dm"
                else [(Species.DARK_MATTER, 0.25, 0), (Species.GAS, 0.75, n ** 3)])
    n_all = n ** 3 * len(lattices)
    ax = torch.arange(n, dtype=torch.float64, device=dev)
    parts = []
    for sp, origin, id0 in lattices:
        axis = origin * d + d * ax
        pos = torch.stack([axis[:, None, None].expand(n, n, n).reshape(-1),
                           axis[None, :, None].expand(n, n, n).reshape(-1),
                           axis[None, None, :].expand(n, n, n).reshape(-1)], dim=1)
        pos += psi.T
        if not bool(torch.isfinite(pos).all()):
            raise ConfigError("non-finite position component")
        pos = pos - L * torch.floor(pos / L)      # wrap_position (box.py)
        pos[pos >= L] -= L
        pos[pos < 0.0] = 0.0
        idx = torch.nonzero(select(pos)).squeeze(1)
        parts.append((sp, idx.cpu().numpy(), pos[idx].cpu().numpy(),
                      (velocity_factor * psi[:, idx]).T.cpu().numpy(), id0))
        del pos
    del psi
    torch.cuda.empty_cache()
    p = ParticleSet(sum(len(x[1]) for x in parts))
    o = 0
    for sp, idx, pos, vel, id0 in parts:
        sl = slice(o, o + len(idx))
        p.pos[sl] = pos
        p.vel[sl] = vel
        p.mass[sl] = box.volume / n_all
        p.species[sl] = sp
        if sp == Species.GAS:
            p.smoothing[sl] = 1.3 * d
            p.internal_energy[sl] = gas_internal_energy
        p.global_id[sl] = idx + id0
        o += len(idx)
    return p


def make_clustered_ic(n_per_dim: int, box: BoxGeometry, seed: int = 0, n_clumps: int = 8,
                      clumped_fraction: float = 0.7,
                      gas_internal_energy: float = 1e-4) -> ParticleSet:
    """Gaussian clumps over a uniform floor, alternating species (hb/ic.py:137-169)."""
    if n_per_dim < 2:
        raise ConfigError("n_per_dim must be >= 2")
    L = box.side_length
    n_total = 2 * n_per_dim ** 3
    rng = np.random.default_rng(seed)
    n_cl = int(clumped_fraction * n_total)
    centers = rng.uniform(0, L, (n_clumps, 3))
    which = rng.integers(0, n_clumps, n_cl)
    clumped = centers[which] + rng.normal(0.0, L / 40.0, (n_cl, 3))
    uniform = rng.uniform(0, L, (n_total - n_cl, 3))
    p = ParticleSet(n_total)
    p.pos = wrap_position(np.vstack([clumped, uniform]), box)
    p.mass[:] = box.volume / n_total
    p.species[:] = np.where(np.arange(n_total) % 2 == 0, np.uint8(Species.DARK_MATTER),
                            np.uint8(Species.GAS))
    gas = p.gas_mask()
    p.smoothing[gas] = 1.3 * (L / (n_total / 2) ** (1.0 / 3.0))
    p.internal_energy[gas] = gas_internal_energy
    p.global_id = np.arange(n_total, dtype=np.int64)
    return p
