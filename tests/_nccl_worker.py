"""Worker for tests/test_gpu_nccl.py (run under torchrun): one DistributedRank
per process over NCCL; two steps; owned-row outputs saved per rank."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(outdir, move=False, drop_ghost=False):
    import torch
    import torch.distributed as dist
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.distributed import DistributedRank, rank_grid_for
    from paper_2510_03557_b200.domain import owner_ranks
    from paper_2510_03557_b200.ic import make_zeldovich_ic
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    box = BoxGeometry(1.0)
    p = make_zeldovich_ic(32, box, 0.3)
    pm = 1.0 / 64
    h = float(p.smoothing.max())
    own = owner_ranks(p.pos, box, rank_grid_for(world)) == rank
    rr = DistributedRank(p.select(np.nonzero(own)[0]), box, rank, world, 2 * pm, 10 * pm,
                         (1.0 / p.n ** (1 / 3)) / 50, h, h, n_global=p.n)
    out, fields = rr.step()
    if move:   # drift every row by up to 0.3 w: migrants cross rank faces
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        d = (torch.rand(fields["pos"].shape, generator=g, device="cuda",
                        dtype=torch.float64) - 0.5) * (0.6 * rr.w)
        fields["pos"] += d
        fields["pos"].remainder_(1.0)
        fields["pos"][fields["pos"] >= 1.0] = 0.0
    if drop_ghost:   # negative control: one shell row loses its mass after the exchange
        rr.exchange()
        f = rr.engine.fields()
        g = torch.nonzero(f["ghost"] != 0)[0, 0] if rank == 0 else None
        if g is not None:
            f["mass"][g] = 0.0
        out = rr.engine.step(rr.passes)
        fields = rr.engine.fields()
        rr.owned_fields = fields
    else:
        out, fields = rr.step()
    torch.cuda.synchronize()
    o = (fields["ghost"] == 0).cpu().numpy()
    res = {"gid": fields["global_id"].cpu().numpy()[o],
           "density": fields["density"].cpu().numpy()[o],
           "pos": fields["pos"].cpu().numpy()[o]}
    for k in ("grav", "hydro", "ncount", "crk_A"):
        res[k] = out[k].cpu().numpy()[:o.size][o]
    # exact in-r_cut source counts of the owned rows (counting pass; it re-steps
    # the rank set, which keeps its leaf order)
    rr.engine.gravity_pair_count()
    counts = rr.engine.out["grav"].reshape(-1).view(torch.int64)[:o.size].cpu().numpy()
    res["gcount"] = counts[o]
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], move="move" in sys.argv[2:], drop_ghost="dropghost" in sys.argv[2:])
