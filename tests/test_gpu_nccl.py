"""GPU, 2 or 4 processes over NCCL (skipped with fewer GPUs): the real
all-to-all overload exchange, which the emulated-rank tests route in-process.
The ranks step twice (move: every row drifts by up to 0.3 overload widths in
between, so migrants change owner through NCCL); their owned rows must equal
one single-domain step of the same set (counts exactly, the rest to FP32
rounding)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,move", [(2, False), (4, False), (2, True), (4, True)])
def test_nccl_ranks_match_single_domain(tmp_path, world, move):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "_nccl_worker.py"), str(tmp_path)] + (["move"] if move else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    got = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(world)]
    merged = {k: np.concatenate([g[k] for g in got]) for k in got[0]}
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    from paper_2510_03557_b200.resident import StepConfig, force_step
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(32, box, 0.3)
    if move:   # the ranks' second step saw the drifted positions: use them
        order = np.argsort(merged["gid"])
        at = np.searchsorted(merged["gid"][order], p.global_id)
        p.pos = merged["pos"][order][at].copy()
    pm = 1.0 / 64
    reach = max(10 * pm, 2 * float(p.smoothing.max()))
    cfg = StepConfig(box=box, bin_width=reach * (1 + 1e-9), max_leaf_size=256, r_s=2 * pm,
                     r_cut=10 * pm, softening=(1.0 / p.n ** (1 / 3)) / 50)
    ref = force_step(p, cfg)
    a, b = np.argsort(merged["gid"]), np.argsort(p.global_id)
    assert merged["gid"].size == p.n
    np.testing.assert_array_equal(merged["gid"][a], p.global_id[b])
    np.testing.assert_array_equal(merged["ncount"][a], ref["ncount"][b])
    for k, refv in (("grav", ref["grav"]), ("hydro", ref["hydro"]), ("crk_A", ref["crk_A"]),
                    ("density", p.density)):
        # FP32 pair sums in different orders: worst particle 1e-4, median 1e-6
        # of the field's scale (a missing pair would be ~1e-3 or more)
        x, y = merged[k][a], refv[b]
        scale = np.abs(y).max()
        err = np.abs(x - y).reshape(len(x), -1).max(axis=1)
        assert err.max() <= 1e-4 * scale, (k, err.max() / scale)
        assert np.median(err) <= 1e-6 * scale, (k, np.median(err) / scale)
