"""Per-sub-phase wall time of the overload exchange under torchrun (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    from bench import _make_rank, make_workload
    from paper_2510_03557_b200.distributed import alltoallv_bytes
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    p, cfg, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
    rr = _make_rank(None, p, cfg, rank, world, meta)
    for _ in range(3):
        rr.step()
    torch.cuda.synchronize()
    h = rr.halo
    T = {}

    def tick(name, t0):
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return time.perf_counter()

    for _ in range(5):
        t = time.perf_counter()
        send, slot_counts, stay, n_stay = h.pack(rr.owned_fields)
        t = tick("pack(select x2 + sync + pack)", t)
        recv, recv_slots = h.route(send, slot_counts)
        t = tick("route (2 NCCL a2a + sync)", t)
        owned_in = int(recv_slots[:, 27].sum())
        new, n_owned = h.unpack(recv, (rr.owned_fields, stay, n_stay), n_stay + owned_in)
        t = tick("unpack (keep gather + sort + unpack)", t)
        rr.engine.set_fields(new, rr.h_range)
        t = tick("set_fields", t)
    if rank == 0:
        print({k: round(v / 5, 3) for k, v in T.items()}, "send MB", send.numel() / 1e6,
              "recv MB", recv.numel() / 1e6, "n", new["pos"].shape[0], "n_stay", n_stay)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
