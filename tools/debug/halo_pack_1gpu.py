"""Single-process timing of one rank's overload pack (hb_halo_pack_all): rank
0 of a `world`-rank decomposition of a config, no communicator needed, so
ncu can wrap it.   python tools/debug/halo_pack_1gpu.py [c4] [4] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch
    from bench import CONFIGS, make_workload
    from paper_2510_03557_b200.distributed import DistributedRank
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    p, cfg, meta = make_workload(cfg_name, 0, world, local=True)
    h = 1.3 * (1.0 / CONFIGS[cfg_name][0])
    rr = DistributedRank(p, cfg.box, 0, world, cfg.r_s, cfg.r_cut, cfg.softening, h, h,
                         cfg.max_leaf_size, n_global=meta["n_particles"])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        send, slots, stay, n_stay = rr.halo.pack(rr.owned_fields)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"pack {ev[0].elapsed_time(ev[1]):.3f} ms, records {send.numel() // rr.halo.rec}, "
              f"n {rr.owned_fields['pos'].shape[0]}, stay {n_stay}", flush=True)


if __name__ == "__main__":
    main()
