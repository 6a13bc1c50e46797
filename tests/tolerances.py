"""FP32-vs-float64 tolerance used by every GPU parity test.

For per-particle vector outputs phi_i = sum_j phi_ij (gravity, hydro, moments)
net values are cancellation residues on near-uniform sets, so the error is
normalised by the reference's own per-particle sum_j |phi_ij| (the bound
hb/lane.py:230-255 reports; SPEC.md:282 uses 8 eps sum|phi|):

    e_i = |phi_i(GPU) - phi_i(ref)| / sum_j |phi_ij|
    median(e) <= 1e-5 and p99.9(e) <= 1e-4,

and on particles whose net value is well conditioned
(|phi_i| >= 1e-2 sum_j|phi_ij|) the plain relative error meets the north-star
bound median <= 1e-5, p99.9 <= 1e-3.
"""
import numpy as np

MED_NORM, P999_NORM = 1e-5, 1e-4
MED_REL, P999_REL = 1e-5, 1e-3


def assert_fp32_close(got, ref, absum, what=""):
    """Raise unless got meets the tolerance; return the error statistics
    {norm_med, norm_p999, rel_med, rel_p999} (rel_* None without conditioned rows)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    absum = np.asarray(absum, dtype=np.float64)
    assert got.shape == ref.shape == absum.shape, (got.shape, ref.shape, absum.shape)
    diff = np.abs(got - ref)
    live = absum > 0
    assert np.all(diff[~live] == 0), f"{what}: nonzero output where the reference has no terms"
    stats = {"norm_med": None, "norm_p999": None, "rel_med": None, "rel_p999": None}
    if not np.any(live):
        return stats
    e = diff[live] / absum[live]
    med, p999 = float(np.median(e)), float(np.quantile(e, 0.999))
    stats.update(norm_med=med, norm_p999=p999)
    assert med <= MED_NORM and p999 <= P999_NORM, f"{what}: normalised med={med:.2e} p99.9={p999:.2e}"
    cond = live & (np.abs(ref) >= 1e-2 * absum)
    if np.any(cond):
        r = diff[cond] / np.abs(ref[cond])
        med, p999 = float(np.median(r)), float(np.quantile(r, 0.999))
        stats.update(rel_med=med, rel_p999=p999)
        assert med <= MED_REL and p999 <= P999_REL, f"{what}: relative med={med:.2e} p99.9={p999:.2e}"
    return stats
