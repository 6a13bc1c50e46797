"""Force evaluation at a PM-interval boundary (the s = 0 boundary of
hb/stepper.py:103-192) and the unordered pair canonicalisation.

The reference's driver path evaluates gravity and hydro in MIRROR mode over
unordered pairs and folds same-rank alias ghosts onto owners; on a rank whose
overload shell holds its own periodic images that double counts pairs across
self-aliased faces (SURVEY.md finding 3).  The GPU engine gathers every
ordered pair on its receiving side instead, which is the reference's own
ordered semantics (hb/lane.py eval_interaction_list, mirror=False) and
counts each physical pair exactly once.
"""
from __future__ import annotations

import numpy as np

from .cmtree import ChainingMesh, InteractionList


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
