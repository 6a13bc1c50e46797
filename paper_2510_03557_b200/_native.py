"""ctypes binding of libhb.so (the C ABI declared in include/hb.h).

This is the only way the package reaches compute: every pair sum, sort, list
and solve runs in the CUDA library.  There is no CPU fallback -- if the
library or a CUDA device is missing, calls raise ``HydroboxError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import HydroboxError, KernelEvalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhb.so")

HB_OK, HB_NONFINITE, HB_OVERFLOW, HB_CONTRACT, HB_CUDA = 0, 1, 2, 3, 4

_lib = None
_lock = threading.Lock()


FIELDSET_ORDER = ("pos", "vel", "mass", "smoothing", "internal_energy", "density", "species",
                  "ghost", "image_shift", "global_id", "ghost_src")


class HbFieldSet(C.Structure):
    """include/hb.h HbFieldSet: SoA rank fields (device pointers)."""
    _fields_ = [(f, C.c_void_p) for f in FIELDSET_ORDER]


def fieldset(fields: dict) -> "HbFieldSet":
    fs = HbFieldSet()
    for f in FIELDSET_ORDER:
        setattr(fs, f, ptr(fields[f]))
    return fs


class HbError(C.Structure):
    _fields_ = [("status", C.c_int32), ("cuda_err", C.c_int32), ("leaf_a", C.c_int64),
                ("leaf_b", C.c_int64), ("msg", C.c_char * 224)]


P = C.c_void_p


class HbMeshArgs(C.Structure):
    _fields_ = [("n", C.c_int64), ("pos", P), ("image_shift", P), ("ghost", P),
                ("side_length", C.c_double), ("lo", C.c_double * 3), ("width", C.c_double * 3),
                ("nb", C.c_int64 * 3), ("max_leaf_size", C.c_int64), ("leaf_cap", C.c_int64),
                ("perm", P), ("leaf_start", P), ("leaf_end", P), ("leaf_lo", P), ("leaf_hi", P),
                ("leaf_ghost_only", P), ("leaf_bin", P), ("bin_ptr", P), ("n_leaves_dev", P),
                ("n_leaves_host", P), ("max_bin_leaves_host", P), ("max_bin_count_host", P)]


class HbListArgs(C.Structure):
    _fields_ = [("n_leaves", C.c_int64), ("leaf_bin", P), ("leaf_lo", P), ("leaf_hi", P),
                ("leaf_level", P), ("leaf_ghost_only", P), ("bin_ptr", P), ("bin_ids", P),
                ("nb", C.c_int64 * 3), ("periodic", C.c_uint8 * 3), ("side_length", C.c_double),
                ("reach", C.c_double), ("active_depth", C.c_int64), ("capacity", C.c_int64),
                ("out_a", P), ("out_b", P), ("out_shift", P), ("count_host", P)]


class HbEvalArgs(C.Structure):
    _fields_ = [("kid", C.c_int32), ("nchan", C.c_int32), ("n", C.c_int64), ("state", P),
                ("pshift", P), ("aux", P), ("naux", C.c_int32), ("W2", C.c_int32),
                ("n_pairs", C.c_int64), ("pair_a", P), ("pair_b", P), ("pair_shift", P),
                ("n_leaves", C.c_int64), ("leaf_start", P), ("leaf_end", P),
                ("params", C.c_double * 4), ("side_length", C.c_double), ("reach", C.c_double),
                ("include_self", C.c_int32), ("mirror", C.c_int32),
                ("chan_sign", C.c_int64 * 10), ("mirror_map", C.c_int64 * 10),
                ("scales", C.c_double * 10), ("deterministic", C.c_int32),
                ("exact_counters", C.c_int32), ("out_int", P), ("out_flt", P),
                ("counters", C.c_int64 * 8)]


def lib():
    """Load libhb.so (built in-tree by __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise HydroboxError(f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
            lb = C.CDLL(LIB_PATH)
            lb.hb_build_mesh_workspace.restype = C.c_size_t
            lb.hb_build_mesh_workspace.argtypes = [C.c_int64, P, C.c_int64]
            lb.hb_leaf_capacity.restype = C.c_int64
            lb.hb_leaf_capacity.argtypes = [C.c_int64, C.c_int64, C.c_int64]
            lb.hb_assemble_lists_workspace.restype = C.c_size_t
            lb.hb_assemble_lists_workspace.argtypes = [C.c_int64, C.c_int64]
            lb.hb_eval_pairs_workspace.restype = C.c_size_t
            lb.hb_eval_pairs_workspace.argtypes = [P]
            for name in ("hb_build_mesh", "hb_assemble_lists", "hb_eval_pairs"):
                getattr(lb, name).argtypes = [P, P, C.c_size_t, P, P]
            lb.hb_permute_rows.argtypes = [C.c_int64, P, P, P, C.c_int64, P, P]
            lb.hb_remap_through_inverse.argtypes = [C.c_int64, P, P, P, P, P]
            lb.hb_grow_aabbs.argtypes = [C.c_int64, P, P, P, P, C.c_double, P, P, P, P]
            lb.hb_launch_count.restype = C.c_int64
            lb.hb_halo_record_bytes.restype = C.c_int64
            lb.hb_halo_select.argtypes = [C.c_int64, P, P, P, C.c_double, C.c_double, C.c_int32,
                                          C.c_int32, C.c_int32, P, P, P, P, P, P, P, P]
            lb.hb_halo_pack.argtypes = [C.c_int64, P, P, P, P, P, P, P, P, P, P, P, C.c_double,
                                        C.c_int32, P, P, P]
            lb.hb_halo_unpack_workspace.restype = C.c_size_t
            lb.hb_halo_unpack_workspace.argtypes = [C.c_int64]
            lb.hb_halo_unpack.argtypes = [C.c_int64, P, C.c_int32, C.c_int64] + [P] * 11 + [
                P, C.c_size_t, P, P]
            lb.hb_halo_resolve_sources.argtypes = [C.c_int64, C.c_int64, P, P, P, P]
            lb.hb_flag_indices_workspace.restype = C.c_size_t
            lb.hb_flag_indices_workspace.argtypes = [C.c_int64]
            lb.hb_flag_indices.argtypes = [C.c_int64, P, P, P, C.c_size_t, P, P]
            lb.hb_crk_solve.argtypes = [C.c_int64, P, C.c_int64, P, C.c_double, P, P, P, P, P]
            lb.hb_timestep_levels.argtypes = [C.c_int64, P, P, P, P, P, C.c_double, C.c_double,
                                              C.c_double, C.c_double, C.c_int64, P, P, P,
                                              C.c_int32, P, P, P, P, P, P]
            lb.hb_pm_deposit.argtypes = [C.c_int64, P, P, C.c_int64, C.c_double, C.c_double, P,
                                         P, P]
            lb.hb_pm_spectral.argtypes = [C.c_int64, C.c_double, C.c_double, P, P, P, P, P, P,
                                          P, P]
            lb.hb_pm_interp.argtypes = [C.c_int64, P, C.c_int32, P, P, P, C.c_int64, C.c_double,
                                        P, P, P]
            lb.hb_fof_workspace.restype = C.c_size_t
            lb.hb_fof_workspace.argtypes = [C.c_int64, C.c_int64 * 3]
            lb.hb_fof_scan.argtypes = [C.c_int64, P, C.c_double * 3, C.c_double * 3,
                                       C.c_int64 * 3, C.c_double, C.c_int32, C.c_double,
                                       C.c_int32, P, P, P, P, P, P, C.c_size_t, P, P]
            lb.hb_uf_union_edges.argtypes = [C.c_int64, P, P, C.c_int64, P, P, P]
            lb.hb_crc32c_device_workspace.restype = C.c_size_t
            lb.hb_crc32c_device_workspace.argtypes = [C.c_int64]
            lb.hb_crc32c_device.argtypes = [P, C.c_int64, P, P, C.c_size_t, P, P]
            lb.hb_crc32c.restype = C.c_uint32
            lb.hb_crc32c.argtypes = [P, C.c_size_t, C.c_uint32]
            lb.hb_halo_pack_all_workspace.restype = C.c_size_t
            lb.hb_halo_pack_all_workspace.argtypes = [C.c_int32]
            lb.hb_halo_pack_all.argtypes = [C.c_int64, C.POINTER(HbFieldSet), C.c_int32 * 3,
                                            C.c_double, C.c_double, C.c_int32, C.c_int32, P, P,
                                            P, C.c_int64, P, P, P, P, C.c_size_t, P, P]
            lb.hb_halo_unpack_keep_workspace.restype = C.c_size_t
            lb.hb_halo_unpack_keep_workspace.argtypes = [C.c_int64, C.c_int64]
            lb.hb_halo_unpack_keep.argtypes = [C.c_int64, P, C.c_int32, C.c_int64,
                                               C.POINTER(HbFieldSet), P, C.c_int64,
                                               C.POINTER(HbFieldSet), P, C.c_size_t, P, P]
            _lib = lb
        return _lib


# every symbol include/hb.h declares (tests check the library exports them)
EXPORTS = ("hb_abi_version", "hb_launch_count", "hb_device_query", "hb_build_mesh_workspace", "hb_leaf_capacity",
           "hb_build_mesh", "hb_permute_rows", "hb_remap_through_inverse", "hb_grow_aabbs",
           "hb_assemble_lists_workspace", "hb_assemble_lists", "hb_eval_pairs_workspace",
           "hb_eval_pairs", "hb_crk_solve", "hb_force_step_workspace", "hb_force_step", "hb_force_step_check", "hb_force_step_workspace_passes",
           "hb_halo_record_bytes", "hb_halo_select", "hb_halo_pack", "hb_halo_unpack_workspace",
           "hb_halo_unpack", "hb_halo_resolve_sources", "hb_halo_pack_all_workspace",
           "hb_halo_pack_all", "hb_halo_unpack_keep_workspace", "hb_halo_unpack_keep",
           "hb_flag_indices_workspace", "hb_flag_indices", "hb_pm_deposit", "hb_pm_spectral",
           "hb_pm_interp", "hb_fof_workspace", "hb_fof_scan", "hb_uf_union_edges", "hb_crc32c",
           "hb_crc32c_device_workspace", "hb_crc32c_device", "hb_timestep_levels")


def torch_cuda():
    """torch with a CUDA device, or a loud failure (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise HydroboxError("no CUDA device: the B200 engine has no CPU fallback")
    return torch


def stream_ptr():
    torch = torch_cuda()
    return P(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> P:
    return P(t.data_ptr()) if t is not None else P(0)


def dev(a, dtype=None):
    """Host numpy (or torch) array -> contiguous CUDA tensor."""
    torch = torch_cuda()
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.cuda()
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if dtype is not None:
        t = t.to(dtype)
    return t.to("cuda", non_blocking=False).contiguous()


def workspace(nbytes: int):
    torch = torch_cuda()
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")


def check(status: int, err: HbError, kernel_name: str | None = None) -> None:
    """Map an HbStatus onto the reference's exception types (hb/errors.py)."""
    if status == HB_OK:
        return
    msg = err.msg.decode(errors="replace")
    if status == HB_NONFINITE and kernel_name is not None:
        raise KernelEvalError(kernel_name,
                              f"non-finite partial in leaf pair ({err.leaf_a}, {err.leaf_b})")
    if status == HB_OVERFLOW and kernel_name is not None:
        raise KernelEvalError(kernel_name,
                              f"accumulator overflow in leaf pair ({err.leaf_a}, {err.leaf_b})")
    raise HydroboxError(f"libhb status {status}: {msg}")
