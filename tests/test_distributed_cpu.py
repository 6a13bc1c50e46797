"""CPU (gloo, world_size 2): the multi-rank plumbing of the overload exchange
-- variable all-to-all of byte records, rank grids and domain bounds."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_03557_b200.distributed import alltoallv_bytes
        rec = 7
        # rank p sends (p + 1) * (r + 1) records to rank r, bytes = p*16 + r
        counts = [(rank + 1) * (r + 1) * rec for r in range(world)]
        send = torch.cat([torch.full((c,), rank * 16 + r, dtype=torch.uint8)
                          for r, c in enumerate(counts)])
        recv, rc = alltoallv_bytes(send, counts)
        expect = torch.cat([torch.full(((p + 1) * (rank + 1) * rec,), p * 16 + rank,
                                       dtype=torch.uint8) for p in range(world)])
        q.put((rank, bool(torch.equal(recv, expect)), rc))
    finally:
        dist.destroy_process_group()


def test_alltoallv_bytes_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    rc = dict((r, c) for r, _, c in res)
    assert rc[0] == [7, 14] and rc[1] == [14, 28]


def test_rank_grid_and_bounds_match_decompose():
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.distributed import domain_bounds, overload_width, rank_grid_for
    from oracle.overload import decompose
    box = BoxGeometry(1.0)
    for world in (1, 2, 4, 8):
        g = rank_grid_for(world)
        assert int(np.prod(g)) == world
        doms = decompose(box, g, 0.1)
        for d in doms:
            lo, hi = domain_bounds(box, g, d.rank_id)
            np.testing.assert_array_equal(lo, d.lo)
            np.testing.assert_array_equal(hi, d.hi)
    # shell: gravity reach or the 2h + 2h density neighbourhood of ghosts in reach
    assert overload_width(5.0, 1.3, headroom=1.0) == pytest.approx(5.2)
    assert overload_width(5.0, 1.0, headroom=1.0) == pytest.approx(5.0)
    with pytest.raises(Exception):
        rank_grid_for(3)
