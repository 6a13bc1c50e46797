"""Python surface of the pair engine (drop-in for hb/lane.py).

``eval_interaction_list`` keeps the reference signature and semantics
(hb/lane.py:122-212): validation and error messages, EvalResult with values,
int64 accumulators in deterministic mode, and the counters dict.  The work is
one hb_eval_pairs call (include/hb.h) on the current CUDA stream; ``lane_width``
only shapes the FLOP-proxy counters and ``workers`` is accepted and ignored
(the GPU schedule replaces the thread pool).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import kernels as K
from .cmtree import ChainingMesh, InteractionList
from .errors import HydroboxError, KernelEvalError
from .kernels import PairKernel


class EvalMode:
    DETERMINISTIC = "deterministic"
    RELAXED = "relaxed"


@dataclass(frozen=True)
class LaneGroup:
    width: int = 8

    def __post_init__(self):
        if self.width < 2 or self.width % 2:
            raise HydroboxError("lane width must be even and >= 2")

    @property
    def half(self) -> int:
        return self.width // 2


@dataclass
class EvalResult:
    values: np.ndarray
    int_acc: np.ndarray | None
    scales: np.ndarray
    counters: dict

    def channel_int_totals(self) -> list[int]:
        if self.int_acc is None:
            raise HydroboxError("integer totals only exist in deterministic mode")
        return [int(sum(int(v) for v in self.int_acc[:, c])) for c in range(self.int_acc.shape[1])]


_STATS: dict[str, dict] = {}


def reset_kernel_stats() -> None:
    _STATS.clear()


def kernel_stats() -> dict[str, dict]:
    return {k: dict(v) for k, v in _STATS.items()}


def _record_stats(kernel: PairKernel, cnt: dict) -> None:
    e = _STATS.setdefault(kernel.name, {"adds": 0, "muls": 0, "fused": 0, "special": 0,
                                        "pairs_scheduled": 0, "pairs_in_reach": 0,
                                        "f_evals": 0, "g_evals": 0, "rotations": 0})
    sched = cnt["pairs_scheduled"]
    c = kernel.op_cost
    e["adds"] += c.adds * sched
    e["muls"] += c.muls * sched
    e["fused"] += c.fmas * sched
    e["special"] += c.special * sched
    for k in ("pairs_scheduled", "pairs_in_reach", "f_evals", "g_evals", "rotations"):
        e[k] += cnt[k]


def eval_on_device(kernel: PairKernel, state_d, pshift_d, aux_d, la_d, lb_d, ls_d, ls_leaf_d,
                   le_leaf_d, n_leaves: int, L: float, deterministic: bool, lane_width: int = 8,
                   mirror: bool = False, out=None, exact_counters: bool = True):
    """Device-level evaluation.  Returns (out tensor, counters dict); `out` is
    accumulated into (allocated zeroed when None)."""
    torch = N.torch_cuda()
    n = int(state_d.shape[0])
    nc = kernel.n_channels
    if out is None:
        out = torch.zeros((n, nc), dtype=torch.int64 if deterministic else torch.float64,
                          device="cuda")
    a = N.HbEvalArgs()
    a.kid, a.nchan, a.n = kernel.kid, nc, n
    a.state, a.pshift = N.ptr(state_d), N.ptr(pshift_d)
    a.aux = N.ptr(aux_d)
    a.naux = int(aux_d.shape[1]) if aux_d is not None else 0
    a.W2 = lane_width // 2
    a.n_pairs = int(la_d.shape[0])
    a.pair_a, a.pair_b, a.pair_shift = N.ptr(la_d), N.ptr(lb_d), N.ptr(ls_d)
    a.n_leaves = int(n_leaves)
    a.leaf_start, a.leaf_end = N.ptr(ls_leaf_d), N.ptr(le_leaf_d)
    for k, v in enumerate(np.asarray(kernel.params, dtype=np.float64)[:4]):
        a.params[k] = float(v)
    a.side_length, a.reach = float(L), float(kernel.reach)
    a.include_self = 1 if kernel.include_self else 0
    a.mirror = 1 if mirror else 0
    for c in range(nc):
        a.chan_sign[c] = int(kernel.channel_signs[c])
        a.mirror_map[c] = int(kernel.mirror_map[c])
        a.scales[c] = float(kernel.scales[c])
    a.deterministic = 1 if deterministic else 0
    a.exact_counters = 1 if exact_counters else 0
    if deterministic:
        a.out_int = N.ptr(out)
    else:
        a.out_flt = N.ptr(out)
    lb = N.lib()
    ws = N.workspace(lb.hb_eval_pairs_workspace(C.byref(a)))
    err = N.HbError()
    st = lb.hb_eval_pairs(C.byref(a), N.ptr(ws), C.c_size_t(ws.numel()), N.stream_ptr(),
                          C.byref(err))
    N.check(st, err, kernel.name)
    c = a.counters
    cdict = {"f_evals": int(c[0]), "g_evals": int(c[1]), "rotations": int(c[2]),
             "pairs_scheduled": int(c[3]), "pairs_in_reach": int(c[4])}
    return out, cdict


def _aux_or_none(aux, n: int, kernel: PairKernel):
    if aux is None:
        if kernel.n_aux:
            raise HydroboxError(f"kernel '{kernel.name}' requires aux columns")
        return None
    aux = np.ascontiguousarray(aux, dtype=np.float64)
    if aux.ndim != 2 or aux.shape[1] < kernel.n_aux:
        raise HydroboxError(f"kernel '{kernel.name}' needs {kernel.n_aux} aux columns")
    return aux


def eval_interaction_list(kernel: PairKernel, ilist: InteractionList, state: np.ndarray,
                          mesh: ChainingMesh, mode: str = EvalMode.DETERMINISTIC,
                          lane_width: int = 8, workers: int = 1, aux: np.ndarray | None = None,
                          mirror: bool = False, pshift: np.ndarray | None = None) -> EvalResult:
    """Evaluate ``kernel`` over every listed leaf pair on the GPU (hb/lane.py:122-212)."""
    if mirror and not kernel.mirrorable:
        raise HydroboxError(f"kernel '{kernel.name}' cannot be mirror-evaluated")
    if kernel.reach > ilist.reach * (1 + 1e-12):
        raise HydroboxError("interaction list was assembled with a smaller reach "
                            f"({ilist.reach:.4g}) than the kernel needs ({kernel.reach:.4g})")
    mirror_map = np.ascontiguousarray(kernel.mirror_map, dtype=np.int64)
    if not np.array_equal(kernel.scales[mirror_map], kernel.scales):
        raise HydroboxError("mirror-swapped channels must share one scale")
    LaneGroup(lane_width)
    torch = N.torch_cuda()
    n = state.shape[0]
    nc = kernel.n_channels
    aux = _aux_or_none(aux, n, kernel)
    det = mode == EvalMode.DETERMINISTIC
    scales = kernel.scales
    empty = {"f_evals": 0, "g_evals": 0, "rotations": 0, "pairs_scheduled": 0,
             "pairs_in_reach": 0}
    if len(ilist) == 0 or n == 0:
        _record_stats(kernel, empty)
        vals = np.zeros((n, nc))
        return EvalResult(vals, np.zeros((n, nc), np.int64) if det else None, scales, empty)
    state_d = N.dev(state, torch.float64)
    pshift_d = N.dev(np.zeros((n, 3), np.int8) if pshift is None else pshift, torch.int8)
    aux_d = N.dev(aux, torch.float64) if aux is not None else None
    out, cdict = eval_on_device(kernel, state_d, pshift_d, aux_d,
                                N.dev(ilist.leaf_a, torch.int64), N.dev(ilist.leaf_b, torch.int64),
                                N.dev(ilist.shift, torch.int8),
                                N.dev(mesh.leaf_start, torch.int64),
                                N.dev(mesh.leaf_end, torch.int64), mesh.n_leaves,
                                mesh.box.side_length, det, lane_width, mirror)
    _record_stats(kernel, cdict)
    if det:
        out_int = out.cpu().numpy()
        if out_int.size and np.abs(out_int).max() >= K.ACC_GUARD:
            raise KernelEvalError(kernel.name, "integer accumulator overflow")
        return EvalResult(out_int.astype(np.float64) / scales, out_int, scales, cdict)
    return EvalResult(out.cpu().numpy(), None, scales, cdict)


def eval_leaf_pair(kernel: PairKernel, leaf_i: int, leaf_j: int, state: np.ndarray,
                   mesh: ChainingMesh, mode: str = EvalMode.DETERMINISTIC, lane_width: int = 8,
                   aux: np.ndarray | None = None, pshift: np.ndarray | None = None) -> np.ndarray:
    """Accumulations of leaf_i's members from one (leaf_i, leaf_j) pair (hb/lane.py:215-227)."""
    ilist = InteractionList(np.array([leaf_i], dtype=np.int64), np.array([leaf_j], dtype=np.int64),
                            kernel.reach, 0)
    res = eval_interaction_list(kernel, ilist, state, mesh, mode=mode, lane_width=lane_width,
                                aux=aux, pshift=pshift)
    s, e = int(mesh.leaf_start[leaf_i]), int(mesh.leaf_end[leaf_i])
    return res.values[s:e]
