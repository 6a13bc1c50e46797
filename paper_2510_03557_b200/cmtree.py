"""Chaining mesh of fixed bins holding shallow k-d leaves -- GPU-built.

Same objects and call contract as hb/cmtree.py (ChainingMesh, Leaf,
InteractionList, build_mesh_and_leaves, grow_bounding_boxes,
assemble_interaction_lists); the work runs in libhb.so
(hb_build_mesh / hb_grow_aabbs / hb_assemble_lists, include/hb.h).  Leaves,
permutation and lists are bit-identical to the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .box import BoxGeometry
from .errors import HydroboxError
from .particles import ParticleSet


@dataclass
class Leaf:
    index: int
    start: int
    end: int
    aabb_lo: np.ndarray
    aabb_hi: np.ndarray
    timestep_level: int
    ghost_only: bool

    @property
    def size(self) -> int:
        return self.end - self.start


@dataclass
class InteractionList:
    """Ordered (receiver, partner, image shift) leaf pairs (hb/cmtree.py:43-63)."""

    leaf_a: np.ndarray
    leaf_b: np.ndarray
    reach: float
    active_depth: int
    shift: np.ndarray = None

    def __post_init__(self):
        if self.shift is None:
            self.shift = np.zeros((self.leaf_a.shape[0], 3), dtype=np.int8)

    def __len__(self) -> int:
        return self.leaf_a.shape[0]


@dataclass
class ChainingMesh:
    box: BoxGeometry
    bounds_lo: np.ndarray
    bounds_hi: np.ndarray
    bin_count: np.ndarray
    bin_width: np.ndarray
    periodic_axis: np.ndarray
    n_particles: int
    leaf_start: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    leaf_end: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    leaf_lo: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    leaf_hi: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    leaf_level: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    leaf_ghost_only: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=bool))
    leaf_bin: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    bin_leaves: list = field(default_factory=list)
    _bin_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.int64))
    _bin_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    _max_bin_leaves: int = 0

    @property
    def n_leaves(self) -> int:
        return self.leaf_start.shape[0]

    def leaf(self, i: int) -> Leaf:
        return Leaf(i, int(self.leaf_start[i]), int(self.leaf_end[i]), self.leaf_lo[i],
                    self.leaf_hi[i], int(self.leaf_level[i]), bool(self.leaf_ghost_only[i]))

    def leaf_of_particle(self) -> np.ndarray:
        sizes = self.leaf_end - self.leaf_start
        return np.repeat(np.arange(self.n_leaves, dtype=np.int64), sizes)

    def max_active_level(self) -> int:
        live = ~self.leaf_ghost_only
        return int(self.leaf_level[live].max()) if np.any(live) else 0


def mesh_geometry(box: BoxGeometry, bin_width: float, bounds_lo=None, bounds_hi=None):
    """Bounds, bins per axis, realised widths, periodic flags (hb/cmtree.py:133-151)."""
    L = box.side_length
    lo = np.zeros(3) if bounds_lo is None else np.asarray(bounds_lo, dtype=np.float64)
    hi = np.full(3, L) if bounds_hi is None else np.asarray(bounds_hi, dtype=np.float64)
    extent = hi - lo
    if np.any(extent <= 0):
        raise HydroboxError("mesh bounds must have positive extent")
    periodic = np.abs(extent - L) < 1e-12 * L
    n_bins = np.maximum(1, np.floor(extent / bin_width).astype(np.int64))
    width = extent / n_bins
    return lo, hi, n_bins, width, periodic


def build_mesh_on_device(pos_d, shift_d, ghost_d, box: BoxGeometry, lo, width, n_bins,
                         max_leaf_size: int):
    """Device-level build: returns dict of device tensors + host counts."""
    torch = N.torch_cuda()
    lb = N.lib()
    n = int(pos_d.shape[0])
    nbins = int(np.prod(n_bins))
    cap = int(lb.hb_leaf_capacity(n, nbins, int(max_leaf_size)))
    nb3 = (C.c_int64 * 3)(*[int(v) for v in n_bins])
    wsz = lb.hb_build_mesh_workspace(n, nb3, int(max_leaf_size))
    ws = N.workspace(wsz)
    out = {
        "perm": torch.empty(max(n, 1), dtype=torch.int64, device="cuda"),
        "leaf_start": torch.empty(cap, dtype=torch.int64, device="cuda"),
        "leaf_end": torch.empty(cap, dtype=torch.int64, device="cuda"),
        "leaf_lo": torch.empty((cap, 3), dtype=torch.float64, device="cuda"),
        "leaf_hi": torch.empty((cap, 3), dtype=torch.float64, device="cuda"),
        "leaf_ghost_only": torch.empty(cap, dtype=torch.uint8, device="cuda"),
        "leaf_bin": torch.empty(cap, dtype=torch.int64, device="cuda"),
        "bin_ptr": torch.empty(nbins + 1, dtype=torch.int64, device="cuda"),
        "n_leaves_dev": torch.zeros(1, dtype=torch.int64, device="cuda"),
    }
    nl = C.c_int64(0)
    mbl = C.c_int64(0)
    a = N.HbMeshArgs()
    a.n = n
    a.pos, a.image_shift, a.ghost = N.ptr(pos_d), N.ptr(shift_d), N.ptr(ghost_d)
    a.side_length = float(box.side_length)
    for d in range(3):
        a.lo[d], a.width[d], a.nb[d] = float(lo[d]), float(width[d]), int(n_bins[d])
    a.max_leaf_size = int(max_leaf_size)
    a.leaf_cap = cap
    for k in ("perm", "leaf_start", "leaf_end", "leaf_lo", "leaf_hi", "leaf_ghost_only",
              "leaf_bin", "bin_ptr", "n_leaves_dev"):
        setattr(a, k, N.ptr(out[k]))
    a.n_leaves_host = C.cast(C.pointer(nl), C.c_void_p)
    a.max_bin_leaves_host = C.cast(C.pointer(mbl), C.c_void_p)
    err = N.HbError()
    st = lb.hb_build_mesh(C.byref(a), N.ptr(ws), C.c_size_t(ws.numel()), N.stream_ptr(),
                          C.byref(err))
    N.check(st, err)
    out["n_leaves"] = int(nl.value)
    out["max_bin_leaves"] = int(mbl.value)
    return out


def build_mesh_and_leaves(particles: ParticleSet, box: BoxGeometry, bin_width: float,
                          max_leaf_size: int, bounds_lo=None, bounds_hi=None) -> ChainingMesh:
    """Build bins and k-d leaves on the GPU and reorder ``particles`` in place
    (hb/cmtree.py:125-196)."""
    lo, hi, n_bins, width, periodic = mesh_geometry(box, bin_width, bounds_lo, bounds_hi)
    mesh = ChainingMesh(box=box, bounds_lo=lo, bounds_hi=hi, bin_count=n_bins, bin_width=width,
                        periodic_axis=periodic, n_particles=particles.n)
    nbins = int(np.prod(n_bins))
    mesh.bin_leaves = [np.zeros(0, dtype=np.int64) for _ in range(nbins)]
    if particles.n == 0:
        mesh._bin_ptr = np.zeros(nbins + 1, dtype=np.int64)
        return mesh
    torch = N.torch_cuda()
    res = build_mesh_on_device(N.dev(particles.pos, torch.float64),
                               N.dev(particles.image_shift, torch.int8),
                               N.dev(particles.ghost, torch.uint8), box, lo, width, n_bins,
                               max_leaf_size)
    nl = res["n_leaves"]
    perm = res["perm"][:particles.n].cpu().numpy()
    particles.apply_permutation(perm)
    mesh.leaf_start = res["leaf_start"][:nl].cpu().numpy()
    mesh.leaf_end = res["leaf_end"][:nl].cpu().numpy()
    mesh.leaf_lo = res["leaf_lo"][:nl].cpu().numpy()
    mesh.leaf_hi = res["leaf_hi"][:nl].cpu().numpy()
    mesh.leaf_ghost_only = res["leaf_ghost_only"][:nl].cpu().numpy().astype(bool)
    mesh.leaf_bin = res["leaf_bin"][:nl].cpu().numpy()
    mesh.leaf_level = np.zeros(nl, dtype=np.int64)
    mesh._bin_ptr = res["bin_ptr"].cpu().numpy()
    mesh._bin_ids = np.arange(nl, dtype=np.int64)
    mesh._max_bin_leaves = res["max_bin_leaves"]
    bp = mesh._bin_ptr
    mesh.bin_leaves = [mesh._bin_ids[bp[b]:bp[b + 1]] for b in range(nbins)]
    return mesh


def grow_bounding_boxes(mesh: ChainingMesh, particles: ParticleSet) -> None:
    """Expand leaf AABBs over current member positions (hb/cmtree.py:199-207)."""
    if mesh.n_leaves == 0:
        return
    torch = N.torch_cuda()
    lo = N.dev(mesh.leaf_lo, torch.float64)
    hi = N.dev(mesh.leaf_hi, torch.float64)
    err = N.HbError()
    st = N.lib().hb_grow_aabbs(
        mesh.n_leaves, N.ptr(N.dev(mesh.leaf_start, torch.int64)),
        N.ptr(N.dev(mesh.leaf_end, torch.int64)), N.ptr(N.dev(particles.pos, torch.float64)),
        N.ptr(N.dev(particles.image_shift, torch.int8)), float(mesh.box.side_length),
        N.ptr(lo), N.ptr(hi), N.stream_ptr(), C.byref(err))
    N.check(st, err)
    mesh.leaf_lo = lo.cpu().numpy()
    mesh.leaf_hi = hi.cpu().numpy()


def check_reach(mesh: ChainingMesh, reach: float) -> None:
    for d in range(3):
        if reach > mesh.bin_width[d] and mesh.bin_count[d] > 3:
            raise HydroboxError(
                f"reach {reach:.4g} exceeds bin width {mesh.bin_width[d]:.4g} on axis {d}")


def assemble_on_device(dev_mesh: dict, n_leaves: int, n_bins, periodic, side_length: float,
                       reach: float, active_depth: int, leaf_level_d=None, bin_ids_d=None):
    """Count + emit the ordered list on device; returns (a, b, shift) tensors."""
    torch = N.torch_cuda()
    lb = N.lib()
    a = N.HbListArgs()
    a.n_leaves = n_leaves
    a.leaf_bin = N.ptr(dev_mesh["leaf_bin"])
    a.leaf_lo = N.ptr(dev_mesh["leaf_lo"])
    a.leaf_hi = N.ptr(dev_mesh["leaf_hi"])
    a.leaf_level = N.ptr(leaf_level_d)
    a.leaf_ghost_only = N.ptr(dev_mesh["leaf_ghost_only"])
    a.bin_ptr = N.ptr(dev_mesh["bin_ptr"])
    a.bin_ids = N.ptr(bin_ids_d)
    for d in range(3):
        a.nb[d] = int(n_bins[d])
        a.periodic[d] = 1 if periodic[d] else 0
    a.side_length = float(side_length)
    a.reach = float(reach)
    a.active_depth = int(active_depth)
    cnt = C.c_int64(0)
    a.count_host = C.cast(C.pointer(cnt), C.c_void_p)
    a.capacity = 0
    err = N.HbError()
    ws = N.workspace(lb.hb_assemble_lists_workspace(n_leaves, 0))
    N.check(lb.hb_assemble_lists(C.byref(a), N.ptr(ws), C.c_size_t(ws.numel()), N.stream_ptr(),
                                 C.byref(err)), err)
    total = int(cnt.value)
    la = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    lbb = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    ls = torch.empty((max(total, 1), 3), dtype=torch.int8, device="cuda")
    if total:
        a.capacity = total
        a.out_a, a.out_b, a.out_shift = N.ptr(la), N.ptr(lbb), N.ptr(ls)
        ws = N.workspace(lb.hb_assemble_lists_workspace(n_leaves, total))
        N.check(lb.hb_assemble_lists(C.byref(a), N.ptr(ws), C.c_size_t(ws.numel()),
                                     N.stream_ptr(), C.byref(err)), err)
    return la[:total], lbb[:total], ls[:total]


def assemble_interaction_lists(mesh: ChainingMesh, reach: float,
                               active_depth: int = 0) -> InteractionList:
    """All (active leaf, partner, image) triples within ``reach``, on the GPU
    (hb/cmtree.py:303-337)."""
    check_reach(mesh, reach)
    active = (mesh.leaf_level >= active_depth) & ~mesh.leaf_ghost_only
    if not np.any(active) or mesh.n_leaves == 0:
        z = np.zeros(0, dtype=np.int64)
        return InteractionList(z, z.copy(), reach, active_depth)
    torch = N.torch_cuda()
    dm = {"leaf_bin": N.dev(mesh.leaf_bin, torch.int64),
          "leaf_lo": N.dev(mesh.leaf_lo, torch.float64),
          "leaf_hi": N.dev(mesh.leaf_hi, torch.float64),
          "leaf_ghost_only": N.dev(mesh.leaf_ghost_only.astype(np.uint8), torch.uint8),
          "bin_ptr": N.dev(mesh._bin_ptr, torch.int64)}
    la, lb, ls = assemble_on_device(dm, mesh.n_leaves, mesh.bin_count, mesh.periodic_axis,
                                    mesh.box.side_length, reach, active_depth,
                                    leaf_level_d=N.dev(mesh.leaf_level, torch.int64),
                                    bin_ids_d=N.dev(mesh._bin_ids, torch.int64))
    return InteractionList(la.cpu().numpy(), lb.cpu().numpy(), reach, active_depth,
                           ls.cpu().numpy())
