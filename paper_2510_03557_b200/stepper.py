"""The PM-interval short-range stepper (hb/stepper.py): the unordered pair
canonicalisation and the device-resident hierarchical subcycle integrator.

The reference's driver path evaluates gravity and hydro in MIRROR mode over
unordered pairs and folds same-rank alias ghosts onto owners; on a rank whose
overload shell holds its own periodic images that double counts pairs across
self-aliased faces (SURVEY.md finding 3).  The GPU engine gathers every
ordered pair on its receiving side instead, which is the reference's own
ordered semantics (hb/lane.py eval_interaction_list, mirror=False) and
counts each physical pair exactly once.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .cmtree import ChainingMesh, InteractionList
from .errors import EnergyError
from .kernels import PairKernel, density_kernel, hydro_force_kernel
from .lane import EvalMode, eval_on_device
from .particles import (COL_CS, COL_H, COL_MASS, COL_P, COL_RHO, COL_SPECIES, COL_VX, COL_X,
                        ParticleSet)


def unordered_due_pairs(ilist: InteractionList, mesh: ChainingMesh):
    """Collapse the ordered list onto canonical unordered (a <= b, shift) entries
    with their pair level (hb/stepper.py:79-100).  Host bookkeeping on the list
    metadata only; the evaluations it feeds run on the GPU."""
    swap = ilist.leaf_a > ilist.leaf_b
    a = np.where(swap, ilist.leaf_b, ilist.leaf_a)
    b = np.where(swap, ilist.leaf_a, ilist.leaf_b)
    sh = np.where(swap[:, None], -ilist.shift, ilist.shift).astype(np.int64)
    same = a == b
    code = (sh[:, 0] * 3 + sh[:, 1]) * 3 + sh[:, 2]
    flip = same & (code < 0)
    sh[flip] *= -1
    key = ((a * mesh.n_leaves + b) * 27 + (sh[:, 0] + 1) * 9 + (sh[:, 1] + 1) * 3 + (sh[:, 2] + 1))
    _, first = np.unique(key, return_index=True)
    a, b, sh = a[first], b[first], sh[first].astype(np.int8)
    level = np.maximum(mesh.leaf_level[a], mesh.leaf_level[b])
    return a, b, sh, level


# ------------------------------------------------------------------ subcycle
# Hierarchical kick-drift-kick over one PM interval: the direct caller of the
# force path (hb/stepper.py:103-192), re-designed to
# stay on the device.  SubcycleEngine keeps the rank's particle fields, leaf
# AABBs / levels and the lists as CUDA tensors for the whole interval; per
# fine boundary it runs the GPU list sweep at the active depth, the density
# pass, the due unordered pairs (canonicalised and bucketed by pair level on
# the device) through hb_eval_pairs in mirror mode, and the kicks / drift as
# fused tensor updates.  Host traffic per boundary: the list and pair counts
# and the momentum / energy checks (a few scalars).
#
# Exact momentum audit (deterministic mode): every listed cross-leaf pair is
# evaluated once and its partner receives the exactly negated quanta by
# integer scatter (hb_eval_pairs deterministic mirror); same-leaf pairs are
# gathered on both sides from one shared FP32 origin, so x_i - x_j and
# x_j - x_i are exact negatives.  The per-boundary quanta sum is therefore 0.



_SUPPORT = 2.0  # spline support radius / h (hb/hydro.py:27)


@dataclass
class ShortRangeContext:
    """Everything the subcycle needs besides the hierarchy (hb/stepper.py:34-50)."""

    particles: ParticleSet
    mesh: ChainingMesh
    box: object
    eos_gamma: float
    reach: float
    mode: str = EvalMode.DETERMINISTIC
    lane_width: int = 8
    workers: int = 1
    gravity_kernel: PairKernel | None = None
    hydro_enabled: bool = True
    visc_alpha: float = 1.0
    visc_beta: float = 2.0


@dataclass
class BoundaryRecord:
    s: int
    depth: int
    kick_scale: float
    pairs_per_level: dict


@dataclass
class SubcycleAudit:
    n_fine: int = 0
    n_boundaries: int = 0
    max_momentum_quanta: int = 0  # max over boundaries and axes of |sum of quanta|
    boundary_log: list = field(default_factory=list)


def exact_column_sums(acc: np.ndarray) -> list:
    """Exact integer column sums (arbitrary precision where int64 could wrap)."""
    if acc.size == 0:
        return [0] * acc.shape[1]
    if int(np.abs(acc).max(initial=0)) < (1 << 62) // max(acc.shape[0], 1):
        return [int(v) for v in acc.sum(axis=0, dtype=np.int64)]
    return [sum(int(v) for v in acc[:, c]) for c in range(acc.shape[1])]


class SubcycleEngine:
    """Device-resident state of one rank for a PM interval of short-range work."""

    FIELDS = ("pos", "vel", "mass", "smoothing", "internal_energy", "density", "species",
              "image_shift", "ghost_src", "accel")

    def __init__(self, ctx: ShortRangeContext):
        torch = N.torch_cuda()
        self.ctx = ctx
        p, mesh = ctx.particles, ctx.mesh
        self.n = p.n
        self.f = {k: N.dev(np.ascontiguousarray(getattr(p, k))) for k in self.FIELDS}
        self.nl = mesh.n_leaves
        self.L = float(mesh.box.side_length)
        self.m = {"leaf_start": N.dev(mesh.leaf_start, torch.int64),
                  "leaf_end": N.dev(mesh.leaf_end, torch.int64),
                  "leaf_lo": N.dev(mesh.leaf_lo, torch.float64),
                  "leaf_hi": N.dev(mesh.leaf_hi, torch.float64),
                  "leaf_level": N.dev(mesh.leaf_level, torch.int64),
                  "leaf_bin": N.dev(mesh.leaf_bin, torch.int64),
                  "leaf_ghost_only": N.dev(mesh.leaf_ghost_only.astype(np.uint8), torch.uint8),
                  "bin_ptr": N.dev(mesh._bin_ptr, torch.int64),
                  "bin_ids": N.dev(mesh._bin_ids, torch.int64)}
        sizes = self.m["leaf_end"] - self.m["leaf_start"]
        self.row_leaf = torch.repeat_interleave(torch.arange(self.nl, device="cuda"), sizes)
        self.gas = self.f["species"] == 1
        self.have_gas = bool(self.gas.any().item())
        alias = torch.nonzero(self.f["ghost_src"] >= 0).flatten()
        self.alias, self.alias_src = alias, self.f["ghost_src"][alias]
        self.det = ctx.mode == EvalMode.DETERMINISTIC

    # -- per-boundary pieces -------------------------------------------------
    def grow(self) -> None:
        err = N.HbError()
        N.check(N.lib().hb_grow_aabbs(
            self.nl, N.ptr(self.m["leaf_start"]), N.ptr(self.m["leaf_end"]),
            N.ptr(self.f["pos"]), N.ptr(self.f["image_shift"]), self.L, N.ptr(self.m["leaf_lo"]),
            N.ptr(self.m["leaf_hi"]), N.stream_ptr(), C.byref(err)), err)

    def lists(self, depth: int):
        from .cmtree import assemble_on_device, check_reach
        mesh = self.ctx.mesh
        check_reach(mesh, self.ctx.reach)
        return assemble_on_device(self.m, self.nl, mesh.bin_count, mesh.periodic_axis, self.L,
                                  self.ctx.reach, depth, leaf_level_d=self.m["leaf_level"],
                                  bin_ids_d=self.m["bin_ids"])

    def state(self):
        """(n,12) float64 engine snapshot (hb/particles.py:135-154) on the device."""
        torch = N.torch_cuda()
        f, g = self.f, self.ctx.eos_gamma
        st = torch.empty((self.n, 12), dtype=torch.float64, device="cuda")
        st[:, COL_X:COL_X + 3] = f["pos"]
        st[:, COL_VX:COL_VX + 3] = f["vel"]
        st[:, COL_MASS] = f["mass"]
        st[:, COL_H] = f["smoothing"]
        self._eos(st)
        st[:, COL_SPECIES] = f["species"].to(torch.float64)
        return st

    def _eos(self, st) -> None:
        torch = N.torch_cuda()
        g, rho, u = self.ctx.eos_gamma, self.f["density"], self.f["internal_energy"]
        st[:, COL_RHO] = rho
        st[:, COL_P] = (g - 1.0) * rho * u
        st[:, COL_CS] = torch.sqrt(torch.clamp(g * (g - 1.0) * u, min=0.0))

    def sync_alias(self, names) -> None:
        if self.alias.numel():
            for k in names:
                self.f[k][self.alias] = self.f[k][self.alias_src]

    def fold_alias(self, acc) -> None:
        if self.alias.numel():
            acc.index_add_(0, self.alias_src, acc[self.alias])
            acc[self.alias] = 0

    def _eval(self, kernel, st, la, lb, ls, mirror: bool):
        out, _ = eval_on_device(kernel, st, self.f["image_shift"], None, la, lb, ls,
                                self.m["leaf_start"], self.m["leaf_end"], self.nl, self.L,
                                self.det, self.ctx.lane_width, mirror=mirror,
                                exact_counters=False)
        return out

    def density(self, st, la, lb, ls, depth: int) -> None:
        """rho over the active list, written back for active gas rows (hb/hydro.py:60-84)."""
        torch = N.torch_cuda()
        h_max = float(self.f["smoothing"].max().item()) if self.n else 0.0
        k = density_kernel(_SUPPORT * h_max)
        out = self._eval(k, st, la, lb, ls, mirror=False)
        rho = (out[:, 0].to(torch.float64) / float(k.scales[0])) if self.det else out[:, 0]
        act_leaf = (self.m["leaf_level"] >= depth) & (self.m["leaf_ghost_only"] == 0)
        rows = act_leaf[self.row_leaf] & self.gas
        self.f["density"] = torch.where(rows, rho, self.f["density"])
        self.sync_alias(("density",))
        self._eos(st)

    def due_pairs(self, la, lb, ls):
        """Canonical unordered (a <= b, shift) pairs and their level (device
        restatement of unordered_due_pairs: the key encodes the pair)."""
        torch = N.torch_cuda()
        sh = ls.to(torch.int64)
        swap = la > lb
        a = torch.where(swap, lb, la)
        b = torch.where(swap, la, lb)
        sh = torch.where(swap[:, None], -sh, sh)
        code = (sh[:, 0] * 3 + sh[:, 1]) * 3 + sh[:, 2]
        sh = torch.where(((a == b) & (code < 0))[:, None], -sh, sh)
        key = (a * self.nl + b) * 27 + (sh[:, 0] + 1) * 9 + (sh[:, 1] + 1) * 3 + (sh[:, 2] + 1)
        key = torch.unique(key, sorted=True)
        c = key % 27
        ab = key // 27
        a, b = ab // self.nl, ab % self.nl
        sh = torch.stack([c // 9 - 1, (c // 3) % 3 - 1, c % 3 - 1], dim=1).to(torch.int8)
        lev = self.m["leaf_level"]
        return a, b, sh, torch.maximum(lev[a], lev[b])

    def impulses(self, st, a, b, sh, h_max: float):
        """[(force (n,3) f64, edot or None, quanta (3,) int64 tensor or None)] of one level."""
        torch = N.torch_cuda()
        ctx, res = self.ctx, []
        kernels = []
        if ctx.gravity_kernel is not None:
            kernels.append((ctx.gravity_kernel, False))
        if ctx.hydro_enabled and self.have_gas:
            kernels.append((hydro_force_kernel(_SUPPORT * h_max, ctx.visc_alpha, ctx.visc_beta),
                            True))
        for k, hydro in kernels:
            acc = self._eval(k, st, a, b, sh, mirror=True)
            self.fold_alias(acc)
            q = acc[:, 0:3].sum(dim=0) if self.det else None
            vals = acc.to(torch.float64) / torch.as_tensor(k.scales, dtype=torch.float64,
                                                          device="cuda") if self.det else acc
            res.append((vals[:, 0:3], vals[:, 3] if hydro else None, q))
        return res

    # -- the interval ----------------------------------------------------------
    def run(self, hierarchy) -> SubcycleAudit:
        torch = N.torch_cuda()
        f = self.f
        nf = hierarchy.n_fine
        dt_fine = hierarchy.dt_pm / nf
        audit = SubcycleAudit(n_fine=nf)
        inv_m = 1.0 / f["mass"]
        for s in range(nf + 1):
            outer = s == 0 or s == nf
            if s > 0:
                self.grow()
            depth = 0 if outer else hierarchy.depth_at(s)
            kick = 0.5 if outer else 1.0
            la, lb, ls = self.lists(depth)
            st = self.state()
            h_max = float(f["smoothing"].max().item()) if self.n else 0.0
            if self.ctx.hydro_enabled and self.have_gas and la.numel():
                self.density(st, la, lb, ls, depth)
            a, b, sh, lev = self.due_pairs(la, lb, ls)
            rec = BoundaryRecord(s=s, depth=depth, kick_scale=kick, pairs_per_level={})
            levels, counts = torch.unique(lev, return_counts=True)
            f_tot, any_kick = None, False
            for m, cnt in zip(levels.tolist(), counts.tolist()):
                rec.pairs_per_level[int(m)] = int(cnt)
                sel = lev == m
                dtk = kick * hierarchy.dt_level(int(m))
                quanta = torch.zeros(3, dtype=torch.int64, device="cuda")
                for force, edot, q in self.impulses(st, a[sel], b[sel], sh[sel], h_max):
                    f["vel"] += force * (dtk * inv_m)[:, None]
                    if edot is not None:
                        f["internal_energy"] += edot * (dtk * inv_m)
                    f_tot = force.clone() if f_tot is None else f_tot + force
                    any_kick = True
                    if q is not None:
                        quanta += q
                audit.max_momentum_quanta = max(audit.max_momentum_quanta,
                                                int(quanta.abs().max().item()))
            if any_kick and depth == 0:  # every pair evaluated: short-range acceleration
                f["accel"] = f_tot * inv_m[:, None]
            if self.ctx.hydro_enabled and self.have_gas:
                umin = float(f["internal_energy"][self.gas].min().item())
                if umin < 0:
                    raise EnergyError("negative internal energy after kick "
                                      f"(min u = {umin:.3e}); timestep too large")
            self.sync_alias(("pos", "vel", "internal_energy", "density", "smoothing", "accel"))
            audit.boundary_log.append(rec)
            audit.n_boundaries += 1
            if s < nf:
                f["pos"] += f["vel"] * dt_fine
                self.sync_alias(("pos", "vel", "internal_energy", "density", "smoothing", "accel"))
        return audit

    def download(self, particles: ParticleSet, mesh: ChainingMesh) -> None:
        for k in ("pos", "vel", "internal_energy", "density", "accel"):
            getattr(particles, k)[...] = self.f[k].cpu().numpy()
        mesh.leaf_lo = self.m["leaf_lo"].cpu().numpy()
        mesh.leaf_hi = self.m["leaf_hi"].cpu().numpy()


def subcycle_pm_step(ctx: ShortRangeContext, hierarchy) -> SubcycleAudit:
    """Advance the rank's particles through one PM interval (hb/stepper.py:103-192):
    upload, SubcycleEngine.run on the device, write the host set back."""
    eng = SubcycleEngine(ctx)
    audit = eng.run(hierarchy)
    eng.download(ctx.particles, ctx.mesh)
    return audit
