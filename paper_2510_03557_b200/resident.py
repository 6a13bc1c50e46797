"""Device-resident force evaluation (the benchmark's hot path).

``ResidentRank`` holds one rank's particle fields as CUDA tensors and runs
``hb_force_step`` (include/hb.h): the s = 0 boundary of subcycle_pm_step
(hb/stepper.py:113-179) -- mesh build + reorder, lists, neighbour count,
density + EOS, CRK moments + solve, short-range gravity, hydro force -- with
the reference's ordered single-count semantics.  Fields ping-pong between two
buffer sets because the build reorders them (the reference reorders its
ParticleSet in place, hb/cmtree.py:171-172).

``force_step(particles, ...)`` is the host-level convenience wrapper: numpy in,
ParticleSet reordered in place, numpy outputs.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .box import BoxGeometry
from .cmtree import mesh_geometry
from .errors import HydroboxError
from .particles import FIELD_SPECS, ParticleSet

PASS_NCOUNT, PASS_DENSITY, PASS_CRK, PASS_GRAVITY, PASS_HYDRO = 1, 2, 4, 8, 16
PASS_ALL = 31
PASS_COUNT_ONLY = 32   # with PASS_GRAVITY: exact in-r_cut source counts, no forces (hb.h)
PASS_CRK_GRAD = 64     # with PASS_CRK: gradA / gradB into out["crk_gradA"], out["crk_gradB"]
PHASES = ("build", "list", "tiling", "sph_density", "sph_force", "gravity", "tail", "total")
KERNELS = ("k_gravity", "k_sph_density", "k_sph_force")  # single-kernel spans (ms_kernel)

STEP_FIELDS = ("pos", "vel", "mass", "smoothing", "internal_energy", "density", "species",
               "ghost", "image_shift", "global_id", "ghost_src")


P = C.c_void_p


class HbStepArgs(C.Structure):
    _fields_ = ([("n", C.c_int64)] + [(f + "_in", P) for f in STEP_FIELDS]
                + [(f, P) for f in STEP_FIELDS]
                + [("side_length", C.c_double), ("lo", C.c_double * 3), ("width", C.c_double * 3),
                   ("nb", C.c_int64 * 3), ("periodic", C.c_uint8 * 3), ("max_leaf_size", C.c_int64),
                   ("reach", C.c_double), ("h_max", C.c_double), ("h_min", C.c_double),
                   ("r_s", C.c_double),
                   ("r_cut", C.c_double), ("softening", C.c_double), ("eos_gamma", C.c_double),
                   ("visc_alpha", C.c_double), ("visc_beta", C.c_double), ("passes", C.c_int32),
                   ("timing", C.c_int32), ("gravity_mode", C.c_int32),
                   ("ghost_density", C.c_int32), ("owned_targets", C.c_int32),
                   ("list_capacity", C.c_int64), ("fields_ready_event", P),
                   ("sph_done_event", P), ("late_fields_event", P),
                   ("perm", P), ("ncount", P), ("grav", P), ("hydro", P), ("crk_moments", P),
                   ("crk_A", P), ("crk_B", P), ("crk_fallback", P), ("n_leaves", C.c_int64),
                   ("n_entries", C.c_int64), ("list_capacity_needed", C.c_int64),
                   ("ms_phase", C.c_float * 8), ("status_out", P), ("ms_kernel", C.c_float * 4),
                   ("crk_moments_out", P), ("grav_half_event", P),
                   ("grav_split_row", C.c_int64), ("crk_gradA", P), ("crk_gradB", P),
                   ("last_fields_event", P)])


def _bind(lib):
    if getattr(lib, "_step_bound", False):
        return
    lib.hb_force_step_workspace.restype = C.c_size_t
    lib.hb_force_step_workspace.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_int64]
    lib.hb_force_step.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    lib.hb_force_step_check.argtypes = [C.c_void_p, C.c_void_p]
    lib.hb_force_step_workspace_passes.restype = C.c_size_t
    lib.hb_force_step_workspace_passes.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                                   C.c_int32]
    lib._step_bound = True


def _event_handle(ev):
    """Raw cudaEvent_t of a torch.cuda.Event (NULL for None).  torch creates
    the CUDA event lazily on its first record(), so an unrecorded event has no
    handle yet: one passed to the step would silently never be recorded."""
    if ev is None:
        return P(0)
    if not ev.cuda_event:
        raise HydroboxError("step event has no CUDA event yet: record() it once first")
    return P(ev.cuda_event)


@dataclass
class StepConfig:
    """Scales of one force evaluation (derived as hb/config.py:79-99 and
    hb/driver.py:121-150 derive them)."""

    box: BoxGeometry
    bin_width: float
    max_leaf_size: int
    r_s: float
    r_cut: float
    softening: float
    eos_gamma: float = 5.0 / 3.0
    visc_alpha: float = 1.0
    visc_beta: float = 2.0
    bounds_lo: np.ndarray | None = None
    bounds_hi: np.ndarray | None = None


class ResidentRank:
    """One rank's working set on the current CUDA device."""

    def __init__(self, particles: ParticleSet | None, cfg: StepConfig, fields: dict | None = None,
                 ghost_density: bool = False, h_range: tuple | None = None,
                 owned_targets: bool = False, gravity_only: bool = False,
                 crk_gradients: bool = False):
        """Either host ``particles`` or device ``fields`` (dict of STEP_FIELDS
        tensors).  ``h_range`` = (h_min_gas, h_max) when given as fields.
        ``owned_targets``: gravity / CRK / hydro outputs are needed for owned
        rows only (ghost rows read 0 in tiles without an owned row)."""
        torch = N.torch_cuda()
        self.cfg = cfg
        self.ghost_density = ghost_density
        self.owned_targets = owned_targets
        lo, hi, nb, width, periodic = mesh_geometry(cfg.box, cfg.bin_width, cfg.bounds_lo,
                                                    cfg.bounds_hi)
        self.lo, self.nb, self.width, self.periodic = lo, nb, width, periodic
        self.lib = N.lib()
        _bind(self.lib)
        self._ws = None
        self._ws_key = None
        self.list_capacity = 0
        self.last = None
        self.out = {}
        self.buf = [None, None]
        # capacity slack for row counts that change between steps (distributed
        # engine); a host-loaded rank keeps its n, so exact capacity
        self._slack = 1.0 if particles is not None else 1.1
        # gravity-only ranks (PASS_GRAVITY, e.g. the dark-matter configs) keep
        # no SPH output buffers
        self.gravity_only = gravity_only
        # gradA / gradB outputs (96 B per row) only when asked for
        self.crk_gradients = crk_gradients and not gravity_only
        if particles is not None:
            gas = particles.species == 1
            h_range = ((float(particles.smoothing[gas].min()), float(particles.smoothing.max()))
                       if np.any(gas) else (0.0, 0.0))
            fields = self._alloc(particles)
        self.set_fields(fields, h_range)

    def set_fields(self, fields: dict, h_range: tuple) -> None:
        """Adopt a device field set (n rows); outputs and the reorder buffer are
        capacity-backed views (no allocation while n stays within capacity)."""
        torch = N.torch_cuda()
        n = int(fields["pos"].shape[0])
        self.h_min, self.h_max = float(h_range[0]), float(h_range[1])
        m = max(n, 1)
        cap = getattr(self, "_cap", 0)
        if m > cap:
            cap = int(m * self._slack) + 1024
            f64 = torch.float64
            self._buf1_store = {k: torch.empty((cap,) + tuple(v.shape[1:]), dtype=v.dtype,
                                               device="cuda") for k, v in fields.items()}
            sph = not self.gravity_only
            self._out_store = {
                "perm": torch.empty(cap, dtype=torch.int64, device="cuda"),
                "grav": torch.zeros((cap, 3), dtype=f64, device="cuda"),
            }
            if sph:
                self._out_store.update({
                    "ncount": torch.zeros(cap, dtype=f64, device="cuda"),
                    "hydro": torch.zeros((cap, 5), dtype=f64, device="cuda"),
                    "crk_A": torch.zeros(cap, dtype=f64, device="cuda"),
                    "crk_B": torch.zeros((cap, 3), dtype=f64, device="cuda"),
                    "crk_fallback": torch.zeros(cap, dtype=torch.uint8, device="cuda"),
                })
            if sph and self.crk_gradients:
                self._out_store.update({
                    "crk_gradA": torch.zeros((cap, 3), dtype=f64, device="cuda"),
                    "crk_gradB": torch.zeros((cap, 3, 3), dtype=f64, device="cuda"),
                })
            self._cap = cap
        self.buf[0] = fields
        self.buf[1] = {k: v[:n] for k, v in self._buf1_store.items()}
        self.cur = 0
        self.out = {k: v[:m] for k, v in self._out_store.items()}
        self.n = n
        nbins = int(np.prod(self.nb))
        leaf_cap = int(self.lib.hb_leaf_capacity(self.n, nbins, self.cfg.max_leaf_size))
        self.list_capacity = max(self.list_capacity, 1024, leaf_cap * 64)

    @staticmethod
    def _alloc(p: ParticleSet) -> dict:
        torch = N.torch_cuda()
        return {name: N.dev(np.ascontiguousarray(getattr(p, name))) for name, _, _ in FIELD_SPECS
                if name in STEP_FIELDS}

    def _workspace(self):
        key = (self._cap, self.list_capacity)
        if self._ws is None or self._ws_key != key:
            nb3 = (C.c_int64 * 3)(*[int(v) for v in self.nb])
            sz = self.lib.hb_force_step_workspace_passes(
                self._cap, nb3, self.cfg.max_leaf_size, self.list_capacity,
                PASS_GRAVITY if self.gravity_only else PASS_ALL)
            if self._ws is None or self._ws.numel() < sz:
                self._ws = None
                self._ws = N.workspace(sz)
            self._ws_key = key
        return self._ws

    def fields(self) -> dict:
        """Current (leaf-ordered after a step) device fields."""
        return self.buf[self.cur]

    def step(self, passes: int = PASS_ALL, timing: bool = False, fields_ready=None,
             sph_done=None, status=None, late_fields=None, grav_half=None,
             last_fields=None) -> dict:
        """One force evaluation; returns the device outputs (leaf order).
        fields_ready / sph_done: optional torch.cuda.Event for copy overlap
        (see HbStepArgs in include/hb.h); late_fields: event after which vel,
        internal_energy, density, global_id and ghost_src are ready (read only from
        the EOS on; fields_ready then covers the rest); last_fields (with
        late_fields, sets without ghost rows only): density, global_id and
        ghost_src are ready, late_fields then covering vel and internal_energy.  status: optional zeroed pinned
        int64[3] tensor; when given (and timing is off) the step returns
        without its final synchronisation and the caller must synchronise the
        stream and call check_status(status) before trusting the outputs."""
        cfg = self.cfg
        src, dst = self.buf[self.cur], self.buf[1 - self.cur]
        a = HbStepArgs()
        a.n = self.n
        for f in STEP_FIELDS:
            setattr(a, f + "_in", N.ptr(src[f]))
            setattr(a, f, N.ptr(dst[f]))
        a.side_length = float(cfg.box.side_length)
        for d in range(3):
            a.lo[d], a.width[d], a.nb[d] = float(self.lo[d]), float(self.width[d]), int(self.nb[d])
            a.periodic[d] = 1 if self.periodic[d] else 0
        a.max_leaf_size = int(cfg.max_leaf_size)
        a.h_max = self.h_max
        a.h_min = self.h_min
        a.reach = max(cfg.r_cut if passes & PASS_GRAVITY else 0.0, 2.0 * self.h_max)
        a.r_s, a.r_cut, a.softening = cfg.r_s, cfg.r_cut, cfg.softening
        a.eos_gamma, a.visc_alpha, a.visc_beta = cfg.eos_gamma, cfg.visc_alpha, cfg.visc_beta
        a.passes = int(passes)
        a.timing = 1 if timing else 0
        a.ghost_density = 1 if self.ghost_density else 0
        a.owned_targets = 1 if self.owned_targets else 0
        a.gravity_mode = int(os.environ.get("HB_GRAVITY_MODE", "0"))
        a.fields_ready_event = _event_handle(fields_ready)
        a.sph_done_event = _event_handle(sph_done)
        a.late_fields_event = _event_handle(late_fields)
        a.last_fields_event = _event_handle(last_fields) if late_fields is not None else P(0)
        a.grav_half_event = _event_handle(grav_half)
        a.status_out = P(status.data_ptr()) if status is not None and not timing else P(0)
        if self.gravity_only and passes & ~(PASS_GRAVITY | PASS_COUNT_ONLY):
            raise HydroboxError("gravity-only rank: SPH passes requested")
        for k in ("perm", "ncount", "grav", "hydro", "crk_A", "crk_B", "crk_fallback",
                  "crk_gradA", "crk_gradB"):
            setattr(a, k, N.ptr(self.out[k]) if k in self.out else P(0))
        if passes & PASS_CRK_GRAD and not (passes & PASS_CRK and "crk_gradA" in self.out):
            raise HydroboxError("PASS_CRK_GRAD needs PASS_CRK and a rank built with "
                                "crk_gradients=True")
        a.crk_moments = P(0)   # moments live in the workspace (include/hb.h)
        for d in range(3):
            if a.reach > self.width[d] and self.nb[d] > 3:
                raise HydroboxError(f"reach {a.reach:.4g} exceeds bin width "
                                    f"{self.width[d]:.4g} on axis {d}")
        for _attempt in range(3):
            ws = self._workspace()
            a.list_capacity = self.list_capacity
            err = N.HbError()
            st = self.lib.hb_force_step(C.byref(a), N.ptr(ws), C.c_size_t(ws.numel()),
                                        N.stream_ptr(), C.byref(err))
            if st == N.HB_CONTRACT and a.list_capacity_needed > self.list_capacity:
                self.list_capacity = int(a.list_capacity_needed * 1.25) + 1024
                continue
            N.check(st, err, "force_step")
            break
        self.cur = 1 - self.cur
        if passes & (PASS_CRK | PASS_HYDRO):
            off = int(a.crk_moments_out or 0) - ws.data_ptr()
            if not 0 <= off <= ws.numel() - self.n * 80:
                raise HydroboxError("force_step placed the CRK moments outside its workspace")
            torch = N.torch_cuda()
            self.out["crk_moments"] = ws[off:off + self.n * 80].view(torch.float64).view(
                self.n, 10)
        self.last = {"n_leaves": int(a.n_leaves), "n_entries": int(a.n_entries),
                     "grav_split_row": int(a.grav_split_row),
                     "ms_phase": ({**dict(zip(PHASES, list(a.ms_phase))),
                                   **dict(zip(KERNELS, list(a.ms_kernel)[:3]))}
                                  if timing else None)}
        return self.out

    def gravity_pair_count(self, owned_only: bool = False) -> int:
        """Exact number of ordered (target, source != target) pairs within
        r_cut over every row (the reference's r2 <= reach2 test with a
        float64 re-check near the threshold, hb/kernels.py:357-359): an
        untimed accounting pass for the FP32 roofline.  Reorders the rank's
        fields like a step does.  owned_only: rows with ghost == 0 only."""
        out = self.step(PASS_GRAVITY | PASS_COUNT_ONLY)
        torch = N.torch_cuda()
        counts = out["grav"].reshape(-1).view(torch.int64)[:self.n]
        if owned_only:
            counts = counts[self.fields()["ghost"] == 0]
        return int(counts.sum().item())

    def check_status(self, status) -> None:
        """Raise the error a deferred step (status=...) recorded; call after
        the step's stream has been synchronised."""
        err = N.HbError()
        N.check(self.lib.hb_force_step_check(P(status.data_ptr()), C.byref(err)), err,
                "force_step")


SPH_OUTPUTS = ("ncount", "crk_A", "crk_B", "hydro")


class HostStepper:
    """End-to-end force evaluation from pinned host arrays (the e2e path).

    Per call: H2D of the 11 input fields in three groups on a copy stream --
    positions/shift/ghost (the mesh build waits only for these), then the
    fields SPH pass A reads, then those first read at the EOS (vel,
    internal_energy, ids) -- the step, and D2H of the results: the SPH
    outputs, density and permutation while gravity is still running, the
    gravity output after.  The step runs with a
    deferred status word, so all copies are enqueued before the host waits;
    the call then synchronises, checks the status and returns host arrays.
    Copies of one call overlap that call's own compute; nothing is carried
    between calls."""

    FIRST = ("pos", "image_shift", "ghost")                  # the mesh build
    EARLY = ("mass", "smoothing", "species")                     # + SPH pass A
    LATE = ("vel", "internal_energy", "density", "global_id", "ghost_src")  # EOS on
    # sets without ghost rows: only vel / internal_energy gate the EOS and
    # pass B; density (non-gas rows), ids and ghost sources are outputs only
    # and land while pass B runs (HbStepArgs.last_fields_event)
    LATE4 = ("vel", "internal_energy")
    LAST4 = ("density", "global_id", "ghost_src")

    def __init__(self, rank: "ResidentRank", pinned_in: dict, pinned_out: dict,
                 passes: int = PASS_ALL):
        torch = N.torch_cuda()
        self.passes = int(passes)
        assert sorted(self.FIRST + self.EARLY + self.LATE) == sorted(STEP_FIELDS)
        assert sorted(self.LATE4 + self.LAST4) == sorted(self.LATE)
        self.rank, self.pin_in, self.pin_out = rank, pinned_in, pinned_out
        self.four_groups = bool(not pinned_in["ghost"].any().item()
                                and not (pinned_in["ghost_src"] >= 0).any().item())
        self.s_in = torch.cuda.Stream()
        self.s_out = torch.cuda.Stream()
        self.ev_first = torch.cuda.Event()
        self.ev_fields = torch.cuda.Event()
        self.ev_sph = torch.cuda.Event()
        self.ev_done = torch.cuda.Event()
        self.ev_late = torch.cuda.Event()
        self.ev_last = torch.cuda.Event()
        self.ev_ghalf = torch.cuda.Event()
        self.status = torch.zeros(3, dtype=torch.int64, pin_memory=True)
        for ev in (self.ev_first, self.ev_fields, self.ev_sph, self.ev_done, self.ev_late,
                   self.ev_last, self.ev_ghalf):
            ev.record()   # materialise the CUDA events (torch creates them lazily)

    def __call__(self):
        torch = N.torch_cuda()
        rk = self.rank
        dst = rk.buf[rk.cur]
        main = torch.cuda.current_stream()
        self.s_in.wait_stream(main)   # previous call's compute may still read dst
        with torch.cuda.stream(self.s_in):
            for f in self.FIRST:
                dst[f].copy_(self.pin_in[f], non_blocking=True)
            self.ev_first.record(self.s_in)
            for f in self.EARLY:
                dst[f].copy_(self.pin_in[f], non_blocking=True)
            self.ev_fields.record(self.s_in)
            for f in (self.LATE4 if self.four_groups else self.LATE):
                dst[f].copy_(self.pin_in[f], non_blocking=True)
            self.ev_late.record(self.s_in)
            if self.four_groups:
                for f in self.LAST4:
                    dst[f].copy_(self.pin_in[f], non_blocking=True)
                self.ev_last.record(self.s_in)
        main.wait_event(self.ev_first)
        self.status.zero_()   # no copy into it is pending: every call ends synchronised
        out = rk.step(self.passes, fields_ready=self.ev_fields, sph_done=self.ev_sph,
                      status=self.status, late_fields=self.ev_late, grav_half=self.ev_ghalf,
                      last_fields=self.ev_last if self.four_groups else None)
        split = rk.last["grav_split_row"]
        self.ev_done.record(main)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_sph)
            for k in SPH_OUTPUTS + ("perm",):
                if k in self.pin_out:
                    self.pin_out[k].copy_(out[k], non_blocking=True)
            if "density" in self.pin_out:
                self.pin_out["density"].copy_(rk.fields()["density"], non_blocking=True)
            self.s_out.wait_event(self.ev_ghalf)   # first gravity half: rows [0, split)
            if split > 0:
                self.pin_out["grav"][:split].copy_(out["grav"][:split], non_blocking=True)
            self.s_out.wait_event(self.ev_done)
            self.pin_out["grav"][split:].copy_(out["grav"][split:], non_blocking=True)
        main.wait_stream(self.s_out)
        main.synchronize()
        rk.check_status(self.status)
        return self.pin_out


def force_step(particles: ParticleSet, cfg: StepConfig, passes: int = PASS_ALL) -> dict:
    """Host-level force evaluation: reorders ``particles`` in place (leaf
    order) and returns numpy outputs; density is updated as compute_density
    updates it."""
    rank = ResidentRank(particles, cfg)
    out = rank.step(passes)
    fields = rank.fields()
    for name in STEP_FIELDS:
        setattr(particles, name, fields[name].cpu().numpy())
    res = {k: v[:particles.n].cpu().numpy() for k, v in out.items()}
    res["crk_fallback"] = res["crk_fallback"].astype(bool)
    res.update(rank.last)
    return res
