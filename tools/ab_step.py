"""A/B timing of the resident force step: per-kernel CUDA-event times over K
steps of one config (median), for the current environment's tuning switches.

    HB_GRAV_JBITS=5 python tools/ab_step.py --config c2 --steps 10
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--tag", default="")
    ap.add_argument("--npd", type=int, default=None, help="lattice override (make_workload npd)")
    args = ap.parse_args()
    import torch
    from bench import make_workload
    from paper_2510_03557_b200.resident import PASS_ALL, PASS_GRAVITY, ResidentRank
    p, cfg, meta = make_workload(args.config, npd=args.npd)
    gonly = meta["n_gas"] == 0
    passes = PASS_GRAVITY if gonly else PASS_ALL
    rr = ResidentRank(p, cfg, gravity_only=gonly)
    for _ in range(3):
        rr.step(passes)
    ph = []
    for _ in range(args.steps):
        rr.step(passes, timing=True)
        ph.append(rr.last["ms_phase"])
    torch.cuda.synchronize()
    med = {k: float(np.median([x[k] for x in ph])) for k in ph[0]}
    env = {k: v for k, v in os.environ.items() if k.startswith("HB_")}
    print(json.dumps({"tag": args.tag, "config": args.config, "env": env, "ms": med}))


if __name__ == "__main__":
    main()
