"""CPU: library loads and exports every symbol of include/hb.h; host-side
logic (geometry, ICs, decomposition, workspace queries) without a GPU."""
import re
import os

import numpy as np
import pytest

from tests.conftest import ROOT


def test_library_exports_header_symbols():
    from paper_2510_03557_b200 import _native
    lib = _native.lib()
    header = open(os.path.join(ROOT, "include", "hb.h")).read()
    declared = set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    for sym in declared:
        getattr(lib, sym)


def test_workspace_queries_are_host_only():
    import ctypes as C
    from paper_2510_03557_b200 import _native as N
    lib = N.lib()
    nb = (C.c_int64 * 3)(25, 25, 25)
    assert lib.hb_build_mesh_workspace(1_000_000, nb, 256) > 24 * 1_000_000
    assert lib.hb_assemble_lists_workspace(10_000, 300_000) > 0
    assert lib.hb_leaf_capacity(1000, 8, 256) >= 8
    a = N.HbEvalArgs()
    a.n, a.n_pairs, a.n_leaves, a.nchan = 10_000, 5_000, 200, 3
    assert lib.hb_eval_pairs_workspace(C.byref(a)) > 10_000 * 16


def test_deferred_status_decoding():
    """hb_force_step_check maps the deferred status words exactly as the
    synchronous end of hb_force_step does (host-only)."""
    import ctypes as C
    from paper_2510_03557_b200 import _native as N
    lib = N.lib()
    lib.hb_force_step_check.argtypes = [C.c_void_p, C.c_void_p]
    ok = 0xFFFFFFFFFFFFFFFF
    cases = [((ok, 0, 0), N.HB_OK), ((ok, 1, 0), N.HB_CONTRACT), ((ok, 0, 1), N.HB_CONTRACT),
             ((4 * 7 + 1, 0, 0), N.HB_NONFINITE), ((4 * 7 + 2, 0, 0), N.HB_OVERFLOW),
             ((0, 0, 0), N.HB_OVERFLOW)]
    for words, want in cases:
        buf = (C.c_uint64 * 3)(*words)
        err = N.HbError()
        assert lib.hb_force_step_check(C.addressof(buf), C.byref(err)) == want, words


def test_rank_local_ic_equals_selection():
    """make_zeldovich_ic(select=...) (bench.py's rank-local workload at N > 1)
    yields exactly the rows a rank would select from the full set."""
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.distributed import rank_grid_for
    from paper_2510_03557_b200.domain import owner_ranks
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    box = BoxGeometry(1.0)
    grid = rank_grid_for(4)
    for sp in ("both", "dm"):
        full = make_zeldovich_ic(16, box, 0.05, species=sp)
        own = owner_ranks(full.pos, box, grid)
        for r in range(4):
            sub = make_zeldovich_ic(16, box, 0.05, species=sp,
                                    select=lambda pos: owner_ranks(pos, box, grid) == r)
            ref = full.select(np.nonzero(own == r)[0])
            for f in ("pos", "vel", "mass", "smoothing", "internal_energy", "density", "species",
                      "ghost", "image_shift", "global_id", "ghost_src", "timestep_level"):
                a, b = getattr(sub, f), getattr(ref, f)
                assert a.dtype == b.dtype and np.array_equal(a, b), (sp, r, f)


def test_leaf_capacity_bounds_the_split():
    from paper_2510_03557_b200 import _native as N
    lib = N.lib()

    def leaves(n, m):
        if n == 0:
            return 0
        if n <= m:
            return 1
        mid = (n + 1) // 2
        return leaves(mid, m) + leaves(n - mid, m)
    rng = np.random.default_rng(0)
    for _ in range(50):
        nbins = int(rng.integers(1, 50))
        m = int(rng.integers(2, 300))
        counts = rng.integers(0, 3000, nbins)
        assert sum(leaves(int(c), m) for c in counts) <= lib.hb_leaf_capacity(int(counts.sum()), nbins, m)


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_03557_b200 import _native
    from paper_2510_03557_b200.errors import HydroboxError
    with pytest.raises(HydroboxError, match="no CPU fallback"):
        _native.torch_cuda()


def test_zeldovich_ic_deterministic_and_normalised():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic, zeldovich_displacement
    box = BoxGeometry(1.0)
    psi = zeldovich_displacement(16, box, 0.05 / 16)
    assert np.isclose(np.sqrt(np.mean(np.sum(psi ** 2, 1))), 0.05 / 16)
    a = make_zeldovich_ic(16, box, 2.0)
    b = make_zeldovich_ic(16, box, 2.0)
    assert np.array_equal(a.pos, b.pos)
    assert a.n == 2 * 16 ** 3 and np.all((a.pos >= 0) & (a.pos < 1))
    assert np.isclose(a.mass.sum(), 1.0)
    # same displacement for both species at their lattice sites
    d = 1 / 16
    n3 = 16 ** 3
    diff = (a.pos[n3:] - a.pos[:n3] - 0.5 * d + 0.5) % 1.0 - 0.5
    assert np.allclose(diff, 0, atol=1e-12)


def test_overload_matches_golden(golden):
    """Host-side overload construction reproduces the reference rank set."""
    from paper_2510_03557_b200.box import BoxGeometry
    from oracle.overload import build_overload, decompose
    from paper_2510_03557_b200.ic import make_lattice_ic
    g = golden("mesh")
    box = BoxGeometry(1.0)
    p = make_lattice_ic(6, box, 0.0, seed=1)
    rs = build_overload(p, decompose(box, (1, 1, 1), 0.3), box, (1, 1, 1))[0][0]
    for f in ("pos", "image_shift", "global_id", "ghost", "ghost_src"):
        np.testing.assert_array_equal(getattr(rs, f), g["lat_in_" + f], err_msg=f)
    p = make_lattice_ic(8, box, 0.02, seed=3)
    rs = build_overload(p, decompose(box, (2, 2, 1), 0.15), box, (2, 2, 1))[0][1]
    for f in ("pos", "image_shift", "global_id", "ghost", "ghost_src"):
        np.testing.assert_array_equal(getattr(rs, f), g["r221_in_" + f], err_msg=f)


def test_unordered_pairs_match_golden(golden):
    from paper_2510_03557_b200.cmtree import InteractionList
    from paper_2510_03557_b200.stepper import unordered_due_pairs
    from tests.conftest import MeshView
    g = golden("lane")
    for c in g["configs"]:
        k = f"c{c}_"
        mesh = MeshView(g, k + "mesh_")
        il = InteractionList(g[k + "la"], g[k + "lb"], 1.0, 0, g[k + "ls"])
        a, b, s, _ = unordered_due_pairs(il, mesh)
        np.testing.assert_array_equal(a, g[k + "ua"])
        np.testing.assert_array_equal(b, g[k + "ub"])
        np.testing.assert_array_equal(s, g[k + "us"])


def test_crc32c_and_catalog_codec_vs_reference(golden):
    """hb_crc32c (host, slice-by-8) against the reference's halo catalog bytes
    (CRC32C footer, hb/insitu.py:371-404) and the CRC32C check value."""
    import struct
    from paper_2510_03557_b200.insitu import crc32c, decode_halo_catalog
    assert crc32c(b"123456789") == 0xE3069283  # CRC-32C check value
    blob = golden("fof")["catalog"].tobytes()
    assert struct.unpack("<I", blob[-4:])[0] == crc32c(blob[:-4])
    assert crc32c(blob[10:], crc32c(blob[:10])) == crc32c(blob)  # running value
    rec = decode_halo_catalog(blob)
    assert rec.shape[0] == 25 and int(rec["step"][0]) == 7


def test_checkpoint_decode_reference_blob(golden):
    """The reference's HCKP blob decodes through the host path (CRCs checked)."""
    from paper_2510_03557_b200.checkpoint import decode_rank_checkpoint
    g = golden("ckpt")
    p, step, rank = decode_rank_checkpoint(g["blob"].tobytes())
    assert (step, rank) == (12, 3)
    for k in ("pos", "vel", "global_id", "ghost_src", "image_shift", "timestep_level"):
        np.testing.assert_array_equal(getattr(p, k), g["in_" + k])


def test_clock_sampler_window():
    """bench.ClockSampler keeps the samples stamped inside the timed window plus
    the nearest one on each side, and reports throttle reasons seen there."""
    import bench
    c = bench.ClockSampler(0)
    rows = [("12:00:00.000", 1965, "Not Active"), ("12:00:00.100", 1900, "Active"),
            ("12:00:00.200", 1950, "Not Active"), ("12:00:05.000", 500, "Not Active")]
    c.lines = [f"2026/10/18 {t}, {mhz}, 1965, Not Active, Not Active, Not Active, {pc}"
               for t, mhz, pc in rows]
    t = bench.ClockSampler._stamp(c.lines[1])
    c.window = [t - 0.01, t + 0.01]
    s = c.summary()
    assert s["samples"] == 3 and s["sm_mhz"] == 1950.0 and s["reasons"] == ["sw_power_cap"]
    c.window = None   # no window: every sample
    assert c.summary()["samples"] == 4


def test_reference_arm_line_contract(capsys):
    """`bench.py --impl reference` at c1 on the host: one JSON line with the
    contract's keys (impl, value/unit, cpu_baseline kind/cores/sample, e2e with
    zero copy bytes)."""
    import argparse
    import json
    import bench
    import time
    args = argparse.Namespace(gpus=1, steps=2, warmup=0, config="c1", impl="reference",
                              cpu_npd=12, no_cpu_baseline=False)
    t0 = time.perf_counter()
    assert bench.run_reference_arm(args) == 0
    wall = time.perf_counter() - t0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["unit"] == bench.UNIT and line["metric"] == bench.METRIC
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": bench.UNIT, "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["config"] == "c1"
    # complete steps, no extrapolation: the timed steps fit the call's wall time
    assert cb["extrapolated"] is False and cb["cpu_model"]
    assert line["steps"] * line["ms_per_step"] * 1e-3 <= wall
    n_up = line["config"]["updates_per_step"]
    assert line["config"]["cpu_sample"]["n_per_dim"] == 12
    assert 0 < n_up < line["config"]["n_particles"]
    assert abs(line["value"] * line["ms_per_step"] * 1e-3 - n_up) <= 1e-6 * n_up
