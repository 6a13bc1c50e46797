"""Run N resident force steps on a config (for ncu launch lists / captures).

    python tools/profile_step.py [--config c2] [--steps 2]
Each step launches, in order: mesh/list/tiling kernels, then k_eval for
ncount, density, crk, gravity, hydro (5 k_eval launches per step)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import torch
    from bench import make_workload
    from paper_2510_03557_b200.resident import ResidentRank
    p, cfg, meta = make_workload(args.config)
    rr = ResidentRank(p, cfg)
    for _ in range(args.steps):
        rr.step(timing=True)
    torch.cuda.synchronize()
    print(rr.last)


if __name__ == "__main__":
    main()
