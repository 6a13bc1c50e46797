"""B200-native short-range particle-particle step of CRK-HACC (arXiv 2510.03557).

Drop-in for the hot path of the reference package `hydrobox`: the same
functions and objects (build_mesh_and_leaves, assemble_interaction_lists,
eval_interaction_list, compute_density, compute_crk_coefficients,
compute_hydro_accel, adapt_smoothing_length, ...), executed by hand-written
sm_100a CUDA kernels in libhb.so behind a C ABI (include/hb.h).
"""
from .box import BoxGeometry, minimum_image, wrap_position
from .cmtree import (ChainingMesh, InteractionList, assemble_interaction_lists,
                     build_mesh_and_leaves, grow_bounding_boxes)
from .errors import HydroboxError, KernelEvalError
from .gravity import ForceSplit, short_range_gravity_kernel
from .hydro import (compute_crk_coefficients, compute_density, compute_hydro_accel,
                    corrected_interpolate, refresh_eos_columns, adapt_smoothing_length)
from .lane import EvalMode, EvalResult, eval_interaction_list
from .particles import ParticleSet, Species

__all__ = [
    "BoxGeometry", "minimum_image", "wrap_position", "ChainingMesh", "InteractionList",
    "assemble_interaction_lists", "build_mesh_and_leaves", "grow_bounding_boxes",
    "HydroboxError", "KernelEvalError", "ForceSplit", "short_range_gravity_kernel",
    "compute_crk_coefficients", "compute_density", "compute_hydro_accel", "corrected_interpolate",
    "refresh_eos_columns", "adapt_smoothing_length", "EvalMode", "EvalResult",
    "eval_interaction_list", "ParticleSet", "Species",
]
