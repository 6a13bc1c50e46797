"""In-situ cluster finding and grid diagnostics (hb/insitu.py; SURVEY.md §8(f)
row 3) on the device.

Friends-of-friends and DBSCAN run rank-locally over owned + ghost rows (image
positions make every cross-boundary edge visible inside some rank), with the
27-stencil cell sweep and a lock-free union-find on the GPU (hb_fof_scan);
rank components are stitched by global id with a second device union over
the (row gid, root gid) edges (hb_uf_union_edges).  Edge decisions use the
reference's float64 expression from the lower row's side, so memberships are
bit-identical to hb/insitu.py.  Group statistics (min-gid halo id, mass,
minimum-image centre of mass, radius) are vectorised segment reductions.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .box import BoxGeometry, minimum_image, wrap_position
from .errors import HydroboxError
from .particles import ParticleSet


@dataclass
class HaloGroup:
    halo_id: int
    member_ids: np.ndarray
    center: np.ndarray
    total_mass: float
    count: int
    radius: float


def _grid_geometry(binpos: np.ndarray, radius: float, box: BoxGeometry, periodic: bool):
    """Cell grid with per-axis width >= radius (hb/insitu.py:142-154)."""
    if periodic:
        lo = np.zeros(3)
        extent = np.full(3, box.side_length)
    else:
        lo = binpos.min(axis=0) - 1e-9
        extent = binpos.max(axis=0) - lo + 2e-9
    ncell = np.maximum(1, np.floor(extent / radius).astype(np.int64))
    inv_w = ncell / extent
    return lo, inv_w, ncell


class _Scanner:
    """One rank set's device positions + cell grid for repeated sweeps."""

    def __init__(self, rs: ParticleSet, box: BoxGeometry, radius: float):
        self.n = rs.n
        self.bare = not np.any(rs.ghost == 1)
        binpos = rs.pos if self.bare else rs.binning_pos(box.side_length)
        self.lo, self.inv_w, self.ncell = _grid_geometry(binpos, radius, box, self.bare)
        self.pos = N.dev(np.ascontiguousarray(binpos, dtype=np.float64))
        self.L = float(box.side_length)
        self.r2 = float(radius * radius)
        nc3 = (C.c_int64 * 3)(*[int(v) for v in self.ncell])
        self.ws = N.workspace(N.lib().hb_fof_workspace(max(self.n, 1), nc3))

    def scan(self, mode, parent=None, core=None, counts=None, border_key=None,
             core_label=None):
        err = N.HbError()
        N.check(N.lib().hb_fof_scan(
            self.n, N.ptr(self.pos), (C.c_double * 3)(*self.lo), (C.c_double * 3)(*self.inv_w),
            (C.c_int64 * 3)(*[int(v) for v in self.ncell]), self.L, 1 if self.bare else 0,
            self.r2, mode, N.ptr(parent), N.ptr(core), N.ptr(counts), N.ptr(border_key),
            N.ptr(core_label), N.ptr(self.ws), C.c_size_t(self.ws.numel()), N.stream_ptr(),
            C.byref(err)), err)

    def components(self, core=None):
        """Row roots (smallest row of each component), mode 0 or core mode 2."""
        torch = N.torch_cuda()
        parent = torch.arange(self.n, dtype=torch.int64, device="cuda")
        self.scan(0 if core is None else 2, parent=parent, core=core)
        return parent


def _as_rank_list(particles) -> list:
    return particles if isinstance(particles, list) else [particles]


def _stitch(edges_a: list, edges_b: list):
    """Union of (gid, gid) edges on the device; returns (unique gids, root gid)."""
    torch = N.torch_cuda()
    a = torch.cat(edges_a)
    b = torch.cat(edges_b)
    uniq, inv = torch.unique(torch.cat([a, b]), return_inverse=True)
    m = a.numel()
    parent = torch.arange(uniq.numel(), dtype=torch.int64, device="cuda")
    err = N.HbError()
    ia, ib = inv[:m].contiguous(), inv[m:].contiguous()
    N.check(N.lib().hb_uf_union_edges(m, N.ptr(ia), N.ptr(ib), uniq.numel(), N.ptr(parent),
                                      N.stream_ptr(), C.byref(err)), err)
    # roots are the smallest dense index = smallest gid (uniq is sorted)
    return uniq, uniq[parent]


def _component_groups(gids: np.ndarray, roots: np.ndarray, pos: np.ndarray, mass: np.ndarray,
                      min_members: int, box: BoxGeometry) -> list:
    """HaloGroup per component with >= min_members (hb/insitu.py:166-189), vectorised:
    halo id = min member gid; centre = wrap(ref + sum m minimage(x - ref) / M)
    about the halo-id member; radius = max |minimage(x - centre)|."""
    if gids.size == 0:
        return []
    if gids.min() >= 0 and roots.min() >= 0 and max(gids.max(), roots.max()) < 2 ** 31:
        # (root, gid) order by one device sort of root << 32 | gid: the same
        # order as np.lexsort((gids, roots)) (gids are unique)
        torch = N.torch_cuda()
        key = torch.from_numpy((roots.astype(np.int64) << 32) | gids.astype(np.int64)).cuda()
        order = torch.argsort(key).cpu().numpy()
    else:
        order = np.lexsort((gids, roots))
    r = roots[order]
    starts = np.flatnonzero(np.r_[True, r[1:] != r[:-1]])
    sizes = np.diff(np.r_[starts, r.size])
    keep = np.flatnonzero(sizes >= min_members)   # only these components become groups
    groups = []
    for s0, sz in zip(starts[keep], sizes[keep]):
        idx = order[s0:s0 + sz]
        members = gids[idx]
        g_x, g_m = pos[idx], mass[idx]
        xm, mm = g_x, g_m
        ref = xm[0]  # members sorted by gid: the min gid (= halo id) comes first
        offs = minimum_image(xm - ref, box)
        total = float(mm.sum())
        center = wrap_position(ref + (mm[:, None] * offs).sum(axis=0) / total, box)
        radius = float(np.linalg.norm(minimum_image(xm - center, box), axis=1).max())
        groups.append(HaloGroup(halo_id=int(members[0]), member_ids=members.astype(np.int64),
                                center=center, total_mass=total, count=int(sz),
                                radius=radius))
    groups.sort(key=lambda q: q.halo_id)
    return groups


def _owned_tables(rank_sets):
    gid, pos, mass = [], [], []
    for rs in rank_sets:
        own = rs.ghost == 0
        gid.append(rs.global_id[own])
        pos.append(rs.pos[own])
        mass.append(rs.mass[own])
    return (np.concatenate(gid).astype(np.int64), np.concatenate(pos), np.concatenate(mass))


def fof_find(particles, box: BoxGeometry, linking_length: float, min_members: int = 10,
             overload_width: float | None = None) -> list:
    """Friends-of-friends groups: connected components of the <= ll pair graph
    (hb/insitu.py:244-270).  ``particles``: one wrapped set (periodic search)
    or a list of overloaded rank sets (plain search + global-id stitching)."""
    N.torch_cuda()  # loud failure without a GPU (no CPU fallback)
    rank_sets = _as_rank_list(particles)
    if overload_width is not None and linking_length > overload_width:
        raise HydroboxError("linking length exceeds overload width: cross-rank "
                            "components are not guaranteed")
    ea, eb = [], []
    for rs in rank_sets:
        sc = _Scanner(rs, box, linking_length)
        roots = sc.components()
        gid = N.dev(np.ascontiguousarray(rs.global_id, dtype=np.int64))
        ea.append(gid)
        eb.append(gid[roots])
    uniq, root = _stitch(ea, eb)
    gids, pos, mass = _owned_tables(rank_sets)
    torch = N.torch_cuda()
    roots = root[torch.searchsorted(uniq, torch.from_numpy(gids).cuda())].cpu().numpy()
    return _component_groups(gids, roots, pos, mass, min_members, box)


def dbscan_find(particles, box: BoxGeometry, eps: float, min_pts: int,
                overload_width: float | None = None):
    """Deterministic DBSCAN (hb/insitu.py:272-368): core points have >= min_pts
    neighbours within eps (self included); clusters are core components; a
    border point joins the adjacent cluster with the lowest label (min core
    gid); the rest is noise.  Returns (groups, noise_gids)."""
    torch = N.torch_cuda()
    rank_sets = _as_rank_list(particles)
    if overload_width is not None and eps > overload_width:
        raise HydroboxError("eps exceeds overload width")
    scans = [_Scanner(rs, box, eps) for rs in rank_sets]
    gid_dev = [N.dev(np.ascontiguousarray(rs.global_id, dtype=np.int64)) for rs in rank_sets]
    # pass 1: neighbour counts -> core gids (owned rows decide)
    core_g = []
    for rs, sc, gd in zip(rank_sets, scans, gid_dev):
        counts = torch.zeros(rs.n, dtype=torch.int64, device="cuda")
        sc.scan(1, counts=counts)
        own = N.dev(rs.ghost == 0)
        core_g.append(gd[own & (counts >= min_pts)])
    core_gids = torch.unique(torch.cat(core_g)) if core_g else torch.zeros(0, dtype=torch.int64)
    # pass 2: core-core components through every rank's view, stitched by gid
    ea, eb, cores = [], [], []
    for rs, sc, gd in zip(rank_sets, scans, gid_dev):
        core = torch.isin(gd, core_gids).to(torch.uint8)
        cores.append(core)
        roots = sc.components(core=core)
        sel = core.bool()
        ea.append(gd[sel])
        eb.append(gd[roots[sel]])
    if core_gids.numel():
        uniq, root = _stitch(ea + [core_gids], eb + [core_gids])
        label = root[torch.searchsorted(uniq, core_gids)]  # cluster label = min core gid
    else:
        label = core_gids
    # pass 3: border attachment by lowest adjacent cluster label
    huge = 2 ** 62
    bg, bl = [], []
    for rs, sc, gd, core in zip(rank_sets, scans, gid_dev, cores):
        core_label = torch.full((rs.n,), huge, dtype=torch.int64, device="cuda")
        if core_gids.numel():
            pos_in = torch.searchsorted(core_gids, gd).clamp(max=core_gids.numel() - 1)
            hit = core_gids[pos_in] == gd
            core_label = torch.where(hit, label[pos_in], core_label)
        border_key = torch.full((rs.n,), huge, dtype=torch.int64, device="cuda")
        sc.scan(3, core=core, border_key=border_key, core_label=core_label)
        own = N.dev(rs.ghost == 0)
        sel = own & (core == 0) & (border_key < huge)
        bg.append(gd[sel])
        bl.append(border_key[sel])
    gids, pos, mass = _owned_tables(rank_sets)
    # core rows take their cluster label (device lookup, same as searchsorted)
    roots_d = torch.full((gids.size,), -1, dtype=torch.int64, device="cuda")
    if core_gids.numel() and gids.size:
        g_d = torch.from_numpy(gids).cuda()
        pos_in = torch.searchsorted(core_gids, g_d).clamp(max=core_gids.numel() - 1)
        roots_d = torch.where(core_gids[pos_in] == g_d, label[pos_in], roots_d)
    roots = roots_d.cpu().numpy()
    if bg:
        b_g = torch.cat(bg).cpu().numpy()
        b_l = torch.cat(bl).cpu().numpy()
        if b_g.size:  # a border gid seen by several ranks: the min label wins
            o = np.lexsort((b_l, b_g))
            b_g, b_l = b_g[o], b_l[o]
            first = np.r_[True, b_g[1:] != b_g[:-1]]
            b_g, b_l = b_g[first], b_l[first]
            where = np.searchsorted(gids, b_g) if np.all(np.diff(gids) > 0) else None
            if where is None:
                gmap = {int(v): k for k, v in enumerate(gids)}
                where = np.array([gmap[int(v)] for v in b_g], dtype=np.int64)
            roots[where] = b_l
    clustered = roots >= 0
    groups = _component_groups(gids[clustered], roots[clustered], pos[clustered],
                               mass[clustered], 1, box)
    noise = np.sort(gids[~clustered]).astype(np.int64)
    return groups, noise


# ------------------------------------------------------------------ catalogs
HCAT_MAGIC = b"HCAT"
HCAT_VERSION = 1
HCAT_SENTINEL = 0x01020304
_HCAT_DTYPE = np.dtype([("halo_id", "<u8"), ("count", "<u8"), ("mass", "<f8"),
                        ("cx", "<f8"), ("cy", "<f8"), ("cz", "<f8"),
                        ("radius", "<f8"), ("step", "<u8")])


def crc32c(data, value: int = 0) -> int:
    """CRC32C (Castagnoli) of a host buffer (hb/crc.py), slice-by-8 in libhb."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8) if isinstance(
        data, (bytes, bytearray, memoryview)) else np.ascontiguousarray(data).view(np.uint8)
    ptr = buf.ctypes.data_as(C.c_void_p) if buf.size else None
    return int(N.lib().hb_crc32c(ptr, C.c_size_t(buf.size), C.c_uint32(value & 0xFFFFFFFF)))


def encode_halo_catalog(groups: list, step: int) -> bytes:
    """Versioned header + records + CRC32C footer (hb/insitu.py:371-384)."""
    rec = np.zeros(len(groups), dtype=_HCAT_DTYPE)
    for i, g in enumerate(sorted(groups, key=lambda q: q.halo_id)):
        rec[i] = (g.halo_id, g.count, g.total_mass, g.center[0], g.center[1], g.center[2],
                  g.radius, step)
    schema = ",".join(_HCAT_DTYPE.names).encode()
    header = HCAT_MAGIC + struct.pack("<IIQH", HCAT_VERSION, HCAT_SENTINEL, len(groups),
                                      len(schema)) + schema
    payload = header + rec.tobytes()
    return payload + struct.pack("<I", crc32c(payload))


def decode_halo_catalog(blob: bytes):
    """Inverse of encode_halo_catalog; validates magic, version, CRC and schema."""
    if blob[:4] != HCAT_MAGIC:
        raise HydroboxError("bad halo catalog magic")
    version, sentinel, count, schema_len = struct.unpack_from("<IIQH", blob, 4)
    if version != HCAT_VERSION or sentinel != HCAT_SENTINEL:
        raise HydroboxError("unsupported halo catalog version or endianness")
    off = 4 + 18
    schema = blob[off:off + schema_len].decode()
    off += schema_len
    body, footer = blob[:-4], blob[-4:]
    if struct.unpack("<I", footer)[0] != crc32c(body):
        raise HydroboxError("halo catalog CRC mismatch")
    if schema != ",".join(_HCAT_DTYPE.names):
        raise HydroboxError("halo catalog schema mismatch")
    return np.frombuffer(body[off:], dtype=_HCAT_DTYPE, count=count)


def halo_catalog_text(groups: list, step: int) -> str:
    lines = ["halo_id\tcount\tmass\tcx\tcy\tcz\tradius\tstep"]
    for g in sorted(groups, key=lambda q: q.halo_id):
        lines.append(f"{g.halo_id}\t{g.count}\t{g.total_mass:.17g}\t{g.center[0]:.17g}\t"
                     f"{g.center[1]:.17g}\t{g.center[2]:.17g}\t{g.radius:.17g}\t{step}")
    return "\n".join(lines) + "\n"


def power_spectrum(density_values, box: BoxGeometry):
    """Binned P(k) of the density contrast on the PM grid (hb/insitu.py:419-443),
    cuFFT on the device: (k centres, P(k), mode counts) without the DC bin."""
    torch = N.torch_cuda()
    rho = density_values if isinstance(density_values, torch.Tensor) else N.dev(
        np.ascontiguousarray(density_values, dtype=np.float64))
    n = int(rho.shape[0])
    rho_bar = float(rho.mean().item())
    if rho_bar <= 0:
        raise HydroboxError("empty density grid")
    dk = torch.fft.fftn(rho / rho_bar - 1.0) / n ** 3
    power = (dk.real ** 2 + dk.imag ** 2).reshape(-1)
    m = torch.from_numpy(np.fft.fftfreq(n) * n).cuda()
    kmag = torch.sqrt(m[:, None, None] ** 2 + m[None, :, None] ** 2 + m[None, None, :] ** 2)
    bins = torch.round(kmag).to(torch.int64).reshape(-1)
    nb = int(bins.max().item()) + 1
    sums = torch.zeros(nb, dtype=torch.float64, device="cuda").index_add_(0, bins, power)
    counts = torch.bincount(bins, minlength=nb)
    pk = torch.where(counts > 0, sums / counts.clamp(min=1), torch.zeros_like(sums)) * box.volume
    kc = 2.0 * np.pi / box.side_length * np.arange(nb)
    return kc[1:], pk.cpu().numpy()[1:], counts.cpu().numpy()[1:]
