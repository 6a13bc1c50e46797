"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Wraps ``_build/liboracle.so`` (hb_oracle.c) with the argument conventions of
the reference API so tests can call ``oracle.eval_pairs(kernel, ...)`` next to
the CUDA product.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline may import this module; the product package never does.

Restated reference functions (hb/ = /root/reference/pkg/src/hydrobox/):
  eval_pairs          hb/lane.py:122-212 (worker chunking, merge order)
  reference_pair_sum  hb/lane.py:230-255
  assemble            hb/cmtree.py:303-337 (+ _assemble_core 210-300)
  build_mesh          hb/cmtree.py:125-196
  crk_solve           hb/hydro.py:115-150
  refresh_eos         hb/hydro.py:48-57
  unordered_due_pairs hb/stepper.py:79-100
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
_lib = None
_lock = threading.Lock()

N_COUNTERS = 8
ACC_GUARD = 2 ** 62


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            _lib = C.CDLL(LIB_PATH)
            _lib.orc_assemble.restype = C.c_int64
            _lib.orc_build_leaves.restype = C.c_int64
            _lib.orc_set_threads.argtypes = [C.c_int]
            _lib.orc_set_threads(os.cpu_count() or 1)
        return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i8(a):
    return np.ascontiguousarray(a, dtype=np.int8)


def eval_pairs(kernel, leaf_a, leaf_b, shift, state, leaf_start, leaf_end, L,
               mode="deterministic", lane_width=8, workers=1, aux=None,
               mirror=False, pshift=None):
    """Restatement of eval_interaction_list (hb/lane.py:122-212).

    Returns (values (n,nc) f64, int_acc or None, counters dict, error kind).
    """
    state = _f64(state)
    n = state.shape[0]
    nc = kernel.n_channels
    if aux is None:
        aux = np.zeros((n, 1))
    aux = _f64(aux)
    if pshift is None:
        pshift = np.zeros((n, 3), np.int8)
    pshift = _i8(pshift)
    leaf_a, leaf_b, shift = _i64(leaf_a), _i64(leaf_b), _i8(shift).reshape(-1, 3)
    npairs = leaf_a.shape[0]
    workers = max(1, min(workers, max(1, npairs)))
    bounds = np.linspace(0, npairs, workers + 1).astype(np.int64)
    det = 1 if mode == "deterministic" else 0
    out_int = np.zeros((n, nc), np.int64)
    out_flt = np.zeros((n, nc))
    counters = np.zeros(N_COUNTERS, np.int64)
    params = _f64(kernel.params)
    sign = _i64(kernel.channel_signs)
    mmap = _i64(kernel.mirror_map)
    scales = _f64(kernel.scales)
    err = lib().orc_eval_pairs_chunked(
        C.c_int(kernel.kid), _p(state), _p(pshift), _p(aux), C.c_int(aux.shape[1]),
        _p(leaf_a), _p(leaf_b), _p(shift), _p(bounds), C.c_int(workers), C.c_int64(n),
        _p(_i64(leaf_start)), _p(_i64(leaf_end)), _p(params), C.c_double(L),
        C.c_int(lane_width // 2), C.c_double(kernel.reach),
        C.c_int(1 if kernel.include_self else 0), C.c_int(1 if mirror else 0),
        _p(sign), _p(mmap), _p(scales), C.c_int(nc), C.c_int(det),
        _p(out_int), _p(out_flt), _p(counters))
    cdict = {"f_evals": int(counters[0]), "g_evals": int(counters[1]),
             "rotations": int(counters[2]), "pairs_scheduled": int(counters[3]),
             "pairs_in_reach": int(counters[4]), "err_kind": int(counters[5]),
             "err_a": int(counters[6]), "err_b": int(counters[7])}
    if det:
        values = out_int.astype(np.float64) / scales
        return values, out_int, cdict, int(err)
    return out_flt, None, cdict, int(err)


def eval_abs_sums(kernel, leaf_a, leaf_b, shift, state, leaf_start, leaf_end, L, aux=None,
                  mirror=False, pshift=None, workers=None):
    """Per-particle sum_j |phi_ij| over the listed pairs (tolerance normaliser)."""
    lib().orc_set_abs_mode(1)
    try:
        vals, _, _, _ = eval_pairs(kernel, leaf_a, leaf_b, shift, state, leaf_start, leaf_end, L,
                                   mode="relaxed", workers=workers or os.cpu_count() or 1,
                                   aux=aux, mirror=mirror, pshift=pshift)
    finally:
        lib().orc_set_abs_mode(0)
    return vals


def reference_pair_sum(kernel, state, L, mode="deterministic", targets=None, aux=None):
    """All-pairs oracle (hb/lane.py:230-255): (values, abs_sums)."""
    state = _f64(state)
    n = state.shape[0]
    nc = kernel.n_channels
    aux = np.zeros((n, 1)) if aux is None else _f64(aux)
    targets = np.arange(n, dtype=np.int64) if targets is None else _i64(targets)
    out_int = np.zeros((n, nc), np.int64)
    out_flt = np.zeros((n, nc))
    out_abs = np.zeros((n, nc))
    det = 1 if mode == "deterministic" else 0
    lib().orc_reference_pairs(
        C.c_int(kernel.kid), _p(state), _p(aux), C.c_int(aux.shape[1]), C.c_int64(n),
        _p(targets), C.c_int64(targets.shape[0]), _p(_f64(kernel.params)), C.c_double(L),
        C.c_double(kernel.reach), C.c_int(1 if kernel.include_self else 0),
        _p(_f64(kernel.scales)), C.c_int(nc), C.c_int(det), _p(out_int), _p(out_flt),
        _p(out_abs))
    if det:
        return out_int.astype(np.float64) / kernel.scales, out_abs
    return out_flt, out_abs


def binning_pos(pos, image_shift, L):
    """pos + shift * L with the reference's two roundings (hb/particles.py:131-133)."""
    return pos + image_shift.astype(np.float64) * L


def mesh_geometry(bounds_lo, bounds_hi, L, bin_width):
    """bins, widths, periodic flags (hb/cmtree.py:144-151)."""
    lo = np.asarray(bounds_lo, dtype=np.float64)
    hi = np.asarray(bounds_hi, dtype=np.float64)
    extent = hi - lo
    periodic = np.abs(extent - L) < 1e-12 * L
    nb = np.maximum(1, np.floor(extent / bin_width).astype(np.int64))
    width = extent / nb
    return lo, hi, nb, width, periodic


def build_mesh(pos, image_shift, ghost, L, bin_width, max_leaf, bounds_lo=None,
               bounds_hi=None):
    """Restated build_mesh_and_leaves: returns a dict with the permutation and
    the columnar leaf arrays (hb/cmtree.py:125-196)."""
    lo = np.zeros(3) if bounds_lo is None else bounds_lo
    hi = np.full(3, L) if bounds_hi is None else bounds_hi
    lo, hi, nb, width, periodic = mesh_geometry(lo, hi, L, bin_width)
    n = pos.shape[0]
    bp = _f64(binning_pos(pos, image_shift, L))
    perm = np.zeros(n, np.int64)
    sizes = np.zeros(max(n, 1), np.int64)
    lbin = np.zeros(max(n, 1), np.int64)
    nl = int(lib().orc_build_leaves(_p(bp), C.c_int64(n), _p(_f64(lo)), _p(_f64(width)),
                                    _p(_i64(nb)), C.c_int64(max_leaf), _p(perm), _p(sizes),
                                    _p(lbin)))
    sizes, lbin = sizes[:nl], lbin[:nl]
    end = np.cumsum(sizes)
    start = end - sizes
    bps = bp[perm]
    if nl:
        llo = np.minimum.reduceat(bps, start, axis=0)
        lhi = np.maximum.reduceat(bps, start, axis=0)
        gsum = np.add.reduceat(np.asarray(ghost)[perm].astype(np.int64), start)
    else:
        llo = np.zeros((0, 3)); lhi = np.zeros((0, 3)); gsum = np.zeros(0, np.int64)
    nbins = int(np.prod(nb))
    counts = np.bincount(lbin, minlength=nbins) if nl else np.zeros(nbins, np.int64)
    bin_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    bin_ids = np.argsort(lbin, kind="stable").astype(np.int64)
    return {"perm": perm, "leaf_start": start, "leaf_end": end, "leaf_lo": llo,
            "leaf_hi": lhi, "leaf_ghost_only": gsum == sizes, "leaf_bin": lbin,
            "bin_count": nb, "bin_width": width, "periodic": periodic, "bounds_lo": lo,
            "bounds_hi": hi, "bin_ptr": bin_ptr, "bin_ids": bin_ids,
            "max_bin_leaves": int(counts.max()) if counts.size else 0}


def assemble(mesh, L, reach, active_depth=0, leaf_level=None):
    """Restated assemble_interaction_lists (hb/cmtree.py:303-337)."""
    nb, width = mesh["bin_count"], mesh["bin_width"]
    for d in range(3):
        if reach > width[d] and nb[d] > 3:
            raise ValueError(f"reach {reach:.4g} exceeds bin width {width[d]:.4g} on axis {d}")
    nl = mesh["leaf_start"].shape[0]
    level = np.zeros(nl, np.int64) if leaf_level is None else np.asarray(leaf_level, np.int64)
    active = (level >= active_depth) & ~np.asarray(mesh["leaf_ghost_only"], bool)
    act = np.nonzero(active)[0].astype(np.int64)
    if act.shape[0] == 0 or nl == 0:
        z = np.zeros(0, np.int64)
        return z, z.copy(), np.zeros((0, 3), np.int8)
    cap = int(act.shape[0]) * 27 * max(1, mesh["max_bin_leaves"])
    oa = np.empty(cap, np.int64); ob = np.empty(cap, np.int64)
    osh = np.empty((cap, 3), np.int8)
    cnt = int(lib().orc_assemble(_p(act), C.c_int64(act.shape[0]), _p(_i64(mesh["leaf_bin"])),
                                 _p(_f64(mesh["leaf_lo"])), _p(_f64(mesh["leaf_hi"])),
                                 _p(_i64(mesh["bin_ptr"])), _p(_i64(mesh["bin_ids"])),
                                 _p(_i64(nb)), _p(np.ascontiguousarray(mesh["periodic"], np.uint8)),
                                 C.c_double(L), C.c_double(reach), _p(oa), _p(ob), _p(osh)))
    la, lb, ls = oa[:cnt], ob[:cnt], osh[:cnt]
    order = np.lexsort((ls[:, 2], ls[:, 1], ls[:, 0], lb, la))
    return la[order], lb[order], ls[order]


def crk_solve(values, gas, cond_limit=1e8):
    """A, B, fallback from the 10 accumulated moments (hb/hydro.py:115-150)."""
    v = values
    n = v.shape[0]
    m0 = v[:, 0]
    m1 = v[:, 1:4].copy()
    m2 = np.empty((n, 3, 3))
    m2[:, 0, 0] = v[:, 4]
    m2[:, 0, 1] = m2[:, 1, 0] = v[:, 5]
    m2[:, 0, 2] = m2[:, 2, 0] = v[:, 6]
    m2[:, 1, 1] = v[:, 7]
    m2[:, 1, 2] = m2[:, 2, 1] = v[:, 8]
    m2[:, 2, 2] = v[:, 9]
    sel = np.asarray(gas, bool) & (m0 > 0)
    A = np.ones(n)
    B = np.zeros((n, 3))
    fb = np.zeros(n, bool)
    idx = np.nonzero(sel)[0]
    if idx.size:
        with np.errstate(all="ignore"):
            cond = np.linalg.cond(m2[idx])
        good = np.isfinite(cond) & (cond < cond_limit)
        fb[idx[~good]] = True
        gi = idx[good]
        if gi.size:
            B[gi] = np.linalg.solve(m2[gi], m1[gi][..., None])[..., 0]
        denom = m0[idx] - np.einsum("ij,ij->i", B[idx], m1[idx])
        bad = ~(np.isfinite(denom) & (np.abs(denom) > 1e-300))
        fb[idx[bad]] = True
        denom[bad] = m0[idx][bad]
        A[idx] = 1.0 / denom
        f = idx[fb[idx]]
        A[f] = 1.0 / m0[f]
        B[f] = 0.0
    return A, B, fb, m0, m1, m2


def refresh_eos(state, density, internal_energy, gamma):
    """P and c_s columns (hb/hydro.py:48-57); modifies state in place."""
    gm1 = gamma - 1.0
    state[:, 8] = density
    state[:, 9] = gm1 * density * internal_energy
    state[:, 10] = np.sqrt(np.maximum(gamma * gm1 * internal_energy, 0.0))


def state_matrix(pos, vel, mass, smoothing, density, internal_energy, species, gamma):
    """(n,12) float64 engine state (hb/particles.py:135-154)."""
    n = pos.shape[0]
    s = np.zeros((n, 12))
    s[:, 0:3] = pos
    s[:, 3:6] = vel
    s[:, 6] = mass
    s[:, 7] = smoothing
    s[:, 8] = density
    gm1 = gamma - 1.0
    s[:, 9] = gm1 * density * internal_energy
    s[:, 10] = np.sqrt(np.maximum(gamma * gm1 * internal_energy, 0.0))
    s[:, 11] = species
    return s


def unordered_due_pairs(la, lb, ls, n_leaves, leaf_level=None):
    """Canonical unordered dedup (hb/stepper.py:79-100)."""
    la, lb = np.asarray(la, np.int64), np.asarray(lb, np.int64)
    swap = la > lb
    a = np.where(swap, lb, la)
    b = np.where(swap, la, lb)
    sh = np.where(swap[:, None], -np.asarray(ls), np.asarray(ls)).astype(np.int64)
    same = a == b
    code = (sh[:, 0] * 3 + sh[:, 1]) * 3 + sh[:, 2]
    flip = same & (code < 0)
    sh[flip] *= -1
    key = ((a * n_leaves + b) * 27 + (sh[:, 0] + 1) * 9 + (sh[:, 1] + 1) * 3 + (sh[:, 2] + 1))
    _, first = np.unique(key, return_index=True)
    a, b, sh = a[first], b[first], sh[first].astype(np.int8)
    if leaf_level is None:
        level = np.zeros(a.shape[0], np.int64)
    else:
        lv = np.asarray(leaf_level)
        level = np.maximum(lv[a], lv[b])
    return a, b, sh, level
