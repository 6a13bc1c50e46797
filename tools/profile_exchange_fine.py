"""Finer wall-time breakdown of one overload exchange under torchrun:
host-side (CPU) time per call and the device drain after it (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    from bench import _make_rank, make_workload
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

    def run(name, fn):
        t0 = time.perf_counter()
        out = fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        a = T.setdefault(name, [0.0, 0.0])
        a[0] += (t1 - t0) * 1e3
        a[1] += (t2 - t1) * 1e3
        return out

    reps = 10
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        send, slot_counts, stay, n_stay = run("pack", lambda: h.pack(rr.owned_fields))
        recv, recv_slots = run("route", lambda: h.route(send, slot_counts))
        owned_in = int(recv_slots[:, 27].sum())
        new, n_owned = run("unpack", lambda: h.unpack(recv, (rr.owned_fields, stay, n_stay),
                                                      n_stay + owned_in))
        run("set_fields", lambda: rr.engine.set_fields(new, rr.h_range))
        out = run("step", lambda: rr.engine.step())
        rr.owned_fields = rr.engine.fields()
    if rank == 0:
        print({k: (round(v[0] / reps, 3), round(v[1] / reps, 3)) for k, v in T.items()},
              "(host ms, device drain ms)", "send MB", send.numel() / 1e6, "n",
              new["pos"].shape[0], "n_stay", n_stay)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
