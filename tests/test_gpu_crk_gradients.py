"""CRK gradient coefficients gradA / gradB (the north star's CRK-SPH gradients;
hb/ has none, so parity is UNPINNED against the reference -- these tests are
the oracle):

* the GPU gradient moments equal a float64 brute-force sum over every
  gas-gas pair within 2 h_i (normalised by the sum of |terms|, FP32 bound);
* known answer: with the corrected kernel W^R_ij = A_i (1 + B_i . dr) W_ij the
  gradient operator sum_j V_j F_j d/dx_i W^R_ij reproduces the gradient of any
  linear field exactly (it is the x_i-derivative of the exact linear
  interpolation identity), so with gradA / gradB it returns grad F to FP32
  accuracy; without them (the plain-kernel gradient) it does not."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIG = 1.0 / math.pi


def _w(q):
    return np.where(q < 1, 1 - 1.5 * q * q + 0.75 * q ** 3, np.where(q < 2, 0.25 * (2 - q) ** 3, 0))


def _gw(q):  # (dw/dq) / q
    qs = np.maximum(q, 1e-30)
    return np.where(q < 1, -3.0 + 2.25 * q, np.where(q < 2, -0.75 * (2 - q) ** 2 / qs, 0))


def _setup():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.hydro import (compute_crk_coefficients, compute_crk_gradients,
                                             compute_density, refresh_eos_columns)
    from paper_2510_03557_b200.ic import make_lattice_ic
    from paper_2510_03557_b200.lane import EvalMode
    box = BoxGeometry(1.0)
    p = make_lattice_ic(10, box, 0.25 / 10, seed=5)
    reach = 2 * float(p.smoothing.max())
    mesh = build_mesh_and_leaves(p, box, max(reach, 1.0 / 3) * (1 + 1e-9), 32)
    il = assemble_interaction_lists(mesh, reach, 0)
    st = p.state_matrix(5 / 3)
    compute_density(p, mesh, st, il, mode=EvalMode.RELAXED)
    refresh_eos_columns(st, p, 5 / 3)
    coeffs = compute_crk_coefficients(p, mesh, st, il, mode=EvalMode.RELAXED)
    grads = compute_crk_gradients(p, mesh, st, il, coeffs)
    return p, coeffs, grads


def _pairs(p):
    """All gas-gas pairs within 2 h_i, minimum image in the unit box (float64)."""
    gas = np.nonzero(p.species == 1)[0]
    x = p.pos[gas]
    dr = x[:, None, :] - x[None, :, :]
    dr -= np.floor(dr + 0.5)
    r = np.sqrt((dr ** 2).sum(-1))
    h = p.smoothing[gas][:, None]
    q = r / h
    V = (p.mass[gas] / p.density[gas])[None, :]
    W = V * SIG / h ** 3 * _w(q)
    G = V * SIG / h ** 5 * _gw(q)
    return gas, dr, W, G


def test_gradient_moments_match_float64():
    p, coeffs, grads = _setup()
    gas, dr, W, G = _pairs(p)
    ref_dm0 = (G[..., None] * dr).sum(1)
    s2 = np.einsum("ij,ija,ijg->iag", G, dr, dr)
    ref_dm1 = -s2 - coeffs.m0[gas][:, None, None] * np.eye(3)
    norm = np.abs(G).sum(1) * np.abs(dr).max()
    e0 = np.abs(grads.dm0[gas] - ref_dm0).max(1) / norm
    e1 = np.abs(grads.dm1[gas] - ref_dm1).max((1, 2)) / (norm * np.abs(dr).max())
    assert np.median(e0) <= 1e-5 and e0.max() <= 1e-4, (np.median(e0), e0.max())
    assert np.median(e1) <= 1e-5 and e1.max() <= 1e-4, (np.median(e1), e1.max())


def test_linear_gradient_reproduction():
    p, coeffs, grads = _setup()
    gas, dr, W, G = _pairs(p)
    A, B = coeffs.A[gas], coeffs.B[gas]
    dA, dB = grads.gradA[gas], grads.gradB[gas]
    g = np.array([1.0, -2.0, 0.5])
    xi = p.pos[gas]
    F = 0.3 + ((xi[:, None, :] - dr) * g).sum(-1)      # F at the image of j seen from i
    lin = 1.0 + np.einsum("ia,ija->ij", B, dr)
    # d/dx_i^g W^R = dA_g lin W + A (dB_ag dr_a + B_g) W + A lin G dr_g
    dWR = (dA[:, None, :] * (lin * W)[..., None]
           + A[:, None, None] * (np.einsum("iag,ija->ijg", dB, dr) + B[:, None, :]) * W[..., None]
           + (A[:, None] * lin * G)[..., None] * dr)
    grad = (F[..., None] * dWR).sum(1)
    ok = ~coeffs.fallback[gas]
    err = np.abs(grad[ok] - g).max(1) / np.abs(g).max()
    assert np.median(err) <= 1e-4 and err.max() <= 1e-3, (np.median(err), err.max())
    # without the coefficient gradients the operator is visibly inexact
    plain = (F[..., None] * (A[:, None] * lin * G)[..., None] * dr).sum(1)
    assert np.median(np.abs(plain[ok] - g).max(1)) > 1e-3


def _resident():
    """The same jittered lattice through the resident step with HB_PASS_CRK_GRAD
    (pass C: gradient moments + the float64 solve in the kernel epilogue)."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_lattice_ic
    from paper_2510_03557_b200.particles import ParticleSet
    from paper_2510_03557_b200.resident import (PASS_ALL, PASS_CRK_GRAD, STEP_FIELDS,
                                                ResidentRank, StepConfig)
    box = BoxGeometry(1.0)
    p = make_lattice_ic(10, box, 0.25 / 10, seed=5)
    reach = 2 * float(p.smoothing.max())
    cfg = StepConfig(box=box, bin_width=max(reach, 1.0 / 3) * (1 + 1e-9), max_leaf_size=32,
                     r_s=0.05, r_cut=0.25, softening=1e-3)
    rr = ResidentRank(p, cfg, crk_gradients=True)
    out = rr.step(PASS_ALL | PASS_CRK_GRAD)
    q = ParticleSet(p.n)
    for f, v in rr.fields().items():
        setattr(q, f, v.cpu().numpy())
    res = {k: out[k][:p.n].cpu().numpy() for k in ("crk_A", "crk_B", "crk_fallback", "crk_gradA",
                                                     "crk_gradB")}
    return q, res


def test_resident_gradients_reproduce_linear_fields():
    """Known answer for the resident pass C: with its gradA / gradB (and its A,
    B, densities) the corrected gradient operator returns grad F of a linear
    field to FP32 accuracy."""
    q, res = _resident()
    gas, dr, W, G = _pairs(q)
    A, B = res["crk_A"][gas], res["crk_B"][gas]
    dA, dB = res["crk_gradA"][gas], res["crk_gradB"][gas]
    g = np.array([1.0, -2.0, 0.5])
    F = 0.3 + ((q.pos[gas][:, None, :] - dr) * g).sum(-1)
    lin = 1.0 + np.einsum("ia,ija->ij", B, dr)
    dWR = (dA[:, None, :] * (lin * W)[..., None]
           + A[:, None, None] * (np.einsum("iag,ija->ijg", dB, dr) + B[:, None, :]) * W[..., None]
           + (A[:, None] * lin * G)[..., None] * dr)
    grad = (F[..., None] * dWR).sum(1)
    ok = ~res["crk_fallback"][gas].astype(bool)
    assert ok.sum() > 0.9 * gas.size
    err = np.abs(grad[ok] - g).max(1) / np.abs(g).max()
    assert np.median(err) <= 1e-4 and err.max() <= 1e-3, (np.median(err), err.max())
    # non-gas rows carry zero gradients
    dm = q.species != 1
    assert not np.any(res["crk_gradA"][dm]) and not np.any(res["crk_gradB"][dm])


def test_resident_gradients_match_compat_path():
    """The resident pass C against the compat path's two gradient-moment passes
    and torch solve (hydro.compute_crk_gradients) on the same leaf-ordered set
    and densities."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.hydro import compute_crk_coefficients, compute_crk_gradients
    from paper_2510_03557_b200.lane import EvalMode
    q, res = _resident()
    reach = 2 * float(q.smoothing.max())
    p = q.copy()
    mesh = build_mesh_and_leaves(p, BoxGeometry(1.0), max(reach, 1.0 / 3) * (1 + 1e-9), 32)
    np.testing.assert_array_equal(p.global_id, q.global_id)    # already in leaf order
    il = assemble_interaction_lists(mesh, reach, 0)
    st = p.state_matrix(5 / 3)
    coeffs = compute_crk_coefficients(p, mesh, st, il, mode=EvalMode.RELAXED)
    grads = compute_crk_gradients(p, mesh, st, il, coeffs)
    gas = p.species == 1
    ok = gas & ~coeffs.fallback
    for k, ref in (("crk_gradA", grads.gradA), ("crk_gradB", grads.gradB)):
        got = res[k][ok].reshape(ok.sum(), -1)
        want = ref[ok].reshape(ok.sum(), -1)
        scale = np.quantile(np.abs(want), 0.99)
        err = np.abs(got - want).max(1) / scale
        assert np.median(err) <= 1e-4 and err.max() <= 1e-2, (k, np.median(err), err.max())
