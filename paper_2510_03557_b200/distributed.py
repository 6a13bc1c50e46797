"""Multi-GPU force evaluation: cuboid ranks with an overload-shell exchange.

One process per GPU.  Each rank owns the particles of one cuboid of the box
(decompose, hb/domain.py:53-69: x-major rank ids, half-open bounds) and, per
step, refreshes its overload shell (refresh_overload / build_overload,
hb/domain.py:88-189) with ONE all-to-all of fixed-width records:

  hb_halo_select (count, emit)   ghost copy for every (rank, image shift) whose
                                 shifted position lies strictly inside the
                                 rank's bounds widened by w; owned copy to the
                                 (new) owner (migration, DriftError on >1 hop)
  hb_halo_pack                   104-byte records, grouped by destination
  all_to_all_single (NCCL)       counts, then bytes (the only collective)
  hb_halo_unpack (+ sort)        owned rows by global_id, ghosts by
                                 (global_id, shift) -- the reference's order
  hb_force_step                  with ghost-only leaves as density receivers,
                                 so ghost rows near the face carry fresh rho,
                                 P, c_s (SURVEY.md finding 4)

The overload width is max(r_cut, 4 h_max) (overload_width()): every ghost
within 2 h_max of an owned particle has its whole density neighbourhood on the
rank, so its rho, P, c_s are fresh.  Results for owned rows equal the
single-domain evaluation within FP32 tolerance.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .box import BoxGeometry
from .errors import DriftError, HydroboxError
from .particles import ParticleSet
from .resident import PASS_ALL, PASS_GRAVITY, STEP_FIELDS, ResidentRank, StepConfig

RANK_GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}

_FIELD_DTYPES = {"pos": ("float64", 3), "vel": ("float64", 3), "mass": ("float64", 1),
                 "smoothing": ("float64", 1), "internal_energy": ("float64", 1),
                 "density": ("float64", 1), "species": ("uint8", 1), "ghost": ("uint8", 1),
                 "image_shift": ("int8", 3), "global_id": ("int64", 1),
                 "ghost_src": ("int64", 1)}


def rank_grid_for(world: int) -> tuple:
    if world in RANK_GRIDS:
        return RANK_GRIDS[world]
    raise HydroboxError(f"no cuboid rank grid for {world} ranks (supported: 1, 2, 4, 8)")


def domain_bounds(box: BoxGeometry, grid, rank: int):
    """Bounds of rank `rank` exactly as decompose() computes them."""
    g = np.asarray(grid, dtype=np.int64)
    L = box.side_length
    c = np.array([rank // (g[1] * g[2]), (rank // g[2]) % g[1], rank % g[2]])
    lo = np.array([L * c[d] / g[d] for d in range(3)])
    hi = np.array([L * (c[d] + 1) / g[d] for d in range(3)])
    return lo, hi


def overload_width(r_cut: float, h_max: float, headroom: float = 1.001) -> float:
    """Smallest valid shell for one evaluation: gravity needs sources within
    r_cut; hydro on an owned particle needs rho, P, c_s of ghosts within
    2 h_max, whose own densities need neighbours within a further 2 h_max.
    (The reference pads 1.25 x reach, hb/driver.py:135-145, for h growth
    between PM-step refreshes; this engine refreshes every evaluation.)"""
    return headroom * max(r_cut, 4.0 * h_max)


def alltoallv_bytes(send, send_counts: list, group=None):
    """Variable all-to-all of a uint8 tensor (NCCL on GPU, gloo on CPU).
    Returns (recv tensor, recv_counts)."""
    import torch
    import torch.distributed as dist
    sc = torch.tensor(send_counts, dtype=torch.int64, device=send.device)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.tolist()]
    out = torch.empty(sum(recv_counts), dtype=torch.uint8, device=send.device)
    dist.all_to_all_single(out, send, recv_counts, [int(x) for x in send_counts], group=group)
    return out, recv_counts


def empty_fields(n: int) -> dict:
    import torch
    out = {}
    for f, (dt, w) in _FIELD_DTYPES.items():
        shape = (n,) if w == 1 else (n, w)
        out[f] = torch.empty(shape, dtype=getattr(torch, dt), device="cuda")
    return out


class HaloExchange:
    """Overload refresh of one rank (world ranks, cuboid grid)."""

    def __init__(self, box: BoxGeometry, grid, w: float, rank: int, world: int, group=None,
                 transport=None, periodic_unsplit: bool = True, n_global: int | None = None):
        self.box, self.grid, self.w = box, tuple(int(x) for x in grid), float(w)
        self.periodic_unsplit = periodic_unsplit
        # key bits of the receiver's (ghost, global_id, shift) sort
        self.key_bits = max(1, int(27 * max(n_global or 2 ** 40, 1) + 26).bit_length())
        self.rank, self.world, self.group = rank, world, group
        self.transport = transport  # callable(send, counts) -> (recv, counts); None = NCCL/gloo
        self.lib = N.lib()
        self.rec = int(self.lib.hb_halo_record_bytes())
        self._bufs = {}   # capacity-backed scratch (no per-step allocation)
        self._sets = [None, None]
        self._which = 0
        lo, hi = domain_bounds(box, self.grid, rank)
        if w >= 0.5 * float(np.min(hi - lo)):
            raise HydroboxError(f"overload_width {w:.4g} >= half the smallest domain extent "
                                f"{float(np.min(hi - lo)):.4g}: a particle would be duplicated "
                                "twice within one rank")

    def _buf(self, name, n, dtype, shape=()):
        import torch
        b = self._bufs.get(name)
        if b is None or b.shape[0] < n:
            b = torch.empty((int(n * 1.2) + 1024,) + tuple(shape), dtype=dtype, device="cuda")
            self._bufs[name] = b
        return b[:n]

    def _field_set(self, n, avoid=None):
        """A capacity-backed rank field set that does not share storage with
        `avoid` (the set being read).  In the step loop the source is the
        engine's own reorder buffer, so one set serves every exchange; the
        second is allocated only if the source is the first (an exchange
        without a step in between)."""
        def alias(cur):
            return (avoid is not None and cur is not None and
                    cur["pos"].untyped_storage().data_ptr() ==
                    avoid["pos"].untyped_storage().data_ptr())
        k = 1 if alias(self._sets[0]) else 0
        cur = self._sets[k]
        if cur is None or cur["pos"].shape[0] < n:
            self._sets[k] = None   # release before allocating the larger set
            cur = empty_fields(int(n * 1.1) + 1024)
            self._sets[k] = cur
        return cur

    @property
    def fast(self) -> bool:
        """Staying owners bypass the exchange.  Valid when no rank can hold a
        periodic self-image of its own particle: unsplit axes periodic in the
        rank mesh and at most 2 ranks along every split axis."""
        return self.periodic_unsplit and all(g <= 2 for g in self.grid)

    def _full(self, name, n, dtype, shape=()):
        """Whole capacity-backed buffer (>= n rows) and its capacity."""
        self._buf(name, n, dtype, shape)
        b = self._bufs[name]
        return b, int(b.shape[0])

    def pack(self, fields: dict):
        """Select + pack in one C call (hb_halo_pack_all: one host sync for the
        counts).  `fields` may be the whole previous rank set: only its owned
        rows (ghost == 0) are sources.  Returns (send bytes, slot counts
        (world, 28) numpy, stay flags or None, number of staying rows)."""
        import torch
        n = int(fields["pos"].shape[0])
        nslot = self.world * 28
        g = (C.c_int32 * 3)(*self.grid)
        counts = self._buf("counts", nslot + 2, torch.int64)
        if getattr(self, "_counts_host", None) is None or self._counts_host.numel() < nslot + 2:
            self._counts_host = torch.zeros(nslot + 2, dtype=torch.int64).pin_memory()
        ch_t = self._counts_host
        stay = self._buf("stay", max(n, 1), torch.uint8) if self.fast else None
        ws = self._buf("pack_ws", int(self.lib.hb_halo_pack_all_workspace(self.world)), torch.uint8)
        fs = N.fieldset(fields)
        pu = 1 if self.periodic_unsplit else 0
        # first call: shell records ~ 6 w / extent of the rows (+ migrants);
        # 8 w / extent, capped at n / 2, avoids a 2x512^3-scale n / 2 buffer
        ext = self.box.side_length / max(self.grid)
        cap = getattr(self, "_rec_cap", max(1024, int(n * min(0.5, 8.0 * self.w / ext))))
        while True:
            rows, cap_r = self._full("rows", cap, torch.int64)
            slots, cap_s = self._full("slots", cap, torch.int32)
            send, cap_b = self._full("send", cap * self.rec, torch.uint8)
            cap = min(cap_r, cap_s, cap_b // self.rec)
            err = N.HbError()
            st = self.lib.hb_halo_pack_all(
                n, C.byref(fs), g, float(self.box.side_length), self.w, self.rank, pu,
                N.ptr(counts), N.ptr(ch_t), N.ptr(stay), cap, N.ptr(rows), N.ptr(slots),
                N.ptr(send), N.ptr(ws), C.c_size_t(ws.numel()), N.stream_ptr(), C.byref(err))
            if st == N.HB_OVERFLOW:
                cap = int(int(ch_t[:nslot].sum()) * 1.25) + 1024
                continue
            N.check(st, err, "halo pack")
            break
        self._rec_cap = cap
        ch_all = ch_t.numpy().copy()
        ch = ch_all[:nslot]
        if int(ch_all[nslot]) & 0xFFFFFFFF:
            raise DriftError("particle crossed more than one domain in one PM step")
        n_stay = int(ch_all[nslot + 1])
        m = int(ch.sum())
        self._counts_dev = counts[:nslot]
        return (send[:m * self.rec], ch.reshape(self.world, 28),
                stay[:n] if stay is not None else None, n_stay)

    def flag_indices(self, flags, count: int, name: str):
        """Row indices of nonzero flags (count known on the host: no sync)."""
        import torch
        n = int(flags.shape[0])
        idx = self._buf(name, max(count, 1), torch.int64)[:count]
        ws = self._buf(name + "_ws", int(self.lib.hb_flag_indices_workspace(n)), torch.uint8)
        err = N.HbError()
        N.check(self.lib.hb_flag_indices(n, N.ptr(flags), N.ptr(idx), N.ptr(ws),
                                         C.c_size_t(ws.numel()), N.stream_ptr(), C.byref(err)),
                err)
        return idx

    def unpack(self, recv, keep=None, n_owned: int | None = None) -> tuple[dict, int]:
        """Records -> new rank field set.  Reference order (keep=None): owned by
        gid then ghosts by (gid, shift).  Fast path keep = (fields, stay, n_stay):
        the staying owned rows first (current order), then arrivals (migrants by
        gid, ghosts by (gid, shift))."""
        import torch
        m = int(recv.numel()) // self.rec
        n0 = int(keep[2]) if keep is not None else 0
        out = self._field_set(max(n0 + m, 1), avoid=keep[0] if keep is not None else None)
        err = N.HbError()
        st = N.stream_ptr()
        if keep is not None:  # staying owned rows (current order), then arrivals: one C call
            src, stay, n_stay = keep
            n_src = int(src["pos"].shape[0])
            ws = self._buf("unpack_ws", int(self.lib.hb_halo_unpack_keep_workspace(n_src, m)),
                           torch.uint8)
            fs_src, fs_dst = N.fieldset(src), N.fieldset(out)
            N.check(self.lib.hb_halo_unpack_keep(m, N.ptr(recv), self.key_bits, n_src,
                                                 C.byref(fs_src), N.ptr(stay), n0,
                                                 C.byref(fs_dst), N.ptr(ws),
                                                 C.c_size_t(ws.numel()), st, C.byref(err)), err)
        else:
            ws = self._buf("unpack_ws", int(self.lib.hb_halo_unpack_workspace(m)), torch.uint8)
            N.check(self.lib.hb_halo_unpack(m, N.ptr(recv), self.key_bits, n0, *[
                N.ptr(out[f]) for f in N.FIELDSET_ORDER], N.ptr(ws), C.c_size_t(ws.numel()), st,
                C.byref(err)), err)
        out = {k: v[:n0 + m] for k, v in out.items()}
        if n_owned is None:
            n_owned = int((out["ghost"] == 0).sum().item())
        if keep is None:
            N.check(self.lib.hb_halo_resolve_sources(n_owned, m, N.ptr(out["global_id"]),
                                                     N.ptr(out["ghost_src"]), st, C.byref(err)),
                    err)
        return out, n_owned

    def route(self, send, slot_counts):
        """All-to-all of the records.  Returns (recv bytes, received slot
        counts (world, 28)).  One host sync (the counts)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return send, slot_counts
        sc = getattr(self, "_counts_dev", None)  # pack's device counts: no H2D copy
        if sc is None or sc.numel() != slot_counts.size:
            sc = torch.from_numpy(np.ascontiguousarray(slot_counts.reshape(-1))).cuda()
        self._counts_dev = None
        rc = self._buf("recv_counts", sc.numel(), torch.int64)
        dist.all_to_all_single(rc, sc, group=self.group)
        recv_slots = rc.cpu().numpy().reshape(self.world, 28)
        send_bytes = [int(x) * self.rec for x in slot_counts.sum(axis=1)]
        recv_bytes = [int(x) * self.rec for x in recv_slots.sum(axis=1)]
        out = self._buf("recv", max(sum(recv_bytes), 1), torch.uint8)[:sum(recv_bytes)]
        dist.all_to_all_single(out, send, recv_bytes, send_bytes, group=self.group)
        return out, recv_slots

    def exchange(self, fields: dict) -> tuple[dict, int]:
        send, slot_counts, stay, n_stay = self.pack(fields)
        if self.transport is not None:
            recv, recv_slots = self.transport(send, slot_counts)
        else:
            recv, recv_slots = self.route(send, slot_counts)
        owned_in = int(np.asarray(recv_slots)[:, 27].sum())
        keep = (fields, stay, n_stay) if stay is not None else None
        return self.unpack(recv, keep, n_stay + owned_in if stay is not None else owned_in)


class DistributedRank:
    """One rank of a multi-GPU force evaluation (device-resident)."""

    def __init__(self, owned: ParticleSet, box: BoxGeometry, rank: int, world: int, r_s: float,
                 r_cut: float, softening: float, h_max: float, h_min: float,
                 max_leaf_size: int = 256, cm_bin_width: float = 0.0, group=None,
                 transport=None, eos_gamma: float = 5.0 / 3.0, periodic_unsplit: bool = True,
                 n_global: int | None = None, passes: int = PASS_ALL):
        import torch
        self.passes = int(passes)
        self.box, self.rank, self.world = box, rank, world
        self.grid = rank_grid_for(world)
        self.w = overload_width(r_cut, h_max)
        reach = max(r_cut, 2.0 * h_max)
        lo, hi = domain_bounds(box, self.grid, rank)
        self.lo, self.hi = lo, hi
        bin_width = max(cm_bin_width, reach * (1 + 1e-9))
        mlo, mhi = lo - self.w, hi + self.w
        if periodic_unsplit:  # unsplit axes: full periodic box, no self-image shell
            for d in range(3):
                if self.grid[d] == 1:
                    mlo[d], mhi[d] = 0.0, box.side_length
        self.cfg = StepConfig(box=box, bin_width=bin_width, max_leaf_size=max_leaf_size,
                              r_s=r_s, r_cut=r_cut, softening=softening, eos_gamma=eos_gamma,
                              bounds_lo=mlo, bounds_hi=mhi)
        self.h_range = (h_min, h_max)
        self.halo = HaloExchange(box, self.grid, self.w, rank, world, group, transport,
                                 periodic_unsplit=periodic_unsplit, n_global=n_global)
        fields = {}
        for f in STEP_FIELDS:
            arr = np.ascontiguousarray(getattr(owned, f))
            fields[f] = torch.from_numpy(arr).cuda()
        fields["ghost"].zero_()
        fields["image_shift"].zero_()
        fields["ghost_src"].fill_(-1)
        self.owned_fields = fields
        self.engine = None
        self.n_owned = int(owned.n)

    def exchange(self):
        new, n_owned = self.halo.exchange(self.owned_fields)
        self.n_owned = n_owned
        self.owned_fields = new   # the rank set holds the owned rows: release the source
        if self.engine is None:
            self.engine = ResidentRank(None, self.cfg, fields=new, ghost_density=self.world > 1,
                                       h_range=self.h_range, owned_targets=self.world > 1,
                                       gravity_only=self.passes == PASS_GRAVITY)
        else:
            self.engine.set_fields(new, self.h_range)
        return new

    def step(self, timing: bool = False, sph_done=None, status=None, grav_half=None):
        """Exchange + force evaluation; returns device outputs (leaf order of
        the rank set) and the reordered fields.  sph_done / status: as
        ResidentRank.step (copy overlap; deferred status, checked with
        self.engine.check_status after the caller's sync)."""
        import torch
        if timing:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        self.exchange()
        if timing:
            e1.record()
        out = self.engine.step(self.passes, timing=timing, sph_done=sph_done, status=status,
                               grav_half=grav_half)
        if timing:
            torch.cuda.synchronize()
            self.engine.last["ms_phase"]["exchange"] = e0.elapsed_time(e1)
        fields = self.engine.fields()
        # next exchange reads the whole rank set: only its owned rows are sources
        self.owned_fields = fields
        return out, fields
