"""Time the pieces of HaloExchange.unpack on one GPU (debug aid)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from bench import make_workload
    from paper_2510_03557_b200 import _native as N
    from paper_2510_03557_b200.distributed import DistributedRank, empty_fields
    from paper_2510_03557_b200.domain import owner_ranks
    p, cfg, meta = make_workload("c2")
    world = 2
    owner = owner_ranks(p.pos, cfg.box, (2, 1, 1))
    gas = p.species == 1
    rr = DistributedRank(p.select(np.nonzero(owner == 0)[0]), cfg.box, 0, world, cfg.r_s,
                         cfg.r_cut, cfg.softening, float(p.smoothing.max()),
                         float(p.smoothing[gas].min()), 256, n_global=p.n)
    h = rr.halo
    send, counts, stay = h.pack(rr.owned_fields)
    recv = send  # rank 0's own view suffices for timing
    lib = N.lib()
    m = recv.numel() // h.rec
    for it in range(3):
        T = {}
        t = time.perf_counter()

        def tick(k):
            nonlocal t
            torch.cuda.synchronize()
            T[k] = (time.perf_counter() - t) * 1e3
            t = time.perf_counter()
        out = empty_fields(m + 10)
        tick("alloc")
        wsz = lib.hb_halo_unpack_workspace(m)
        tick("ws query")
        ws = N.workspace(wsz)
        tick("ws alloc")
        err = N.HbError()
        N.check(lib.hb_halo_unpack(m, N.ptr(recv), h.key_bits, 0, *[N.ptr(out[f]) for f in (
            "pos", "vel", "mass", "smoothing", "internal_energy", "density", "species", "ghost",
            "image_shift", "global_id", "ghost_src")], N.ptr(ws), C.c_size_t(ws.numel()),
            N.stream_ptr(), C.byref(err)), err)
        tick("unpack kernel+sort")
        n_owned = int((out["ghost"] == 0).sum().item())
        tick("count")
        print(it, m, wsz / 1e6, "MB ws", {k: round(v, 3) for k, v in T.items()}, h.key_bits)


if __name__ == "__main__":
    main()
