"""A small resident force step (2x16^3 Zel'dovich, every pass, plus the
counting pass and the compat pair engine) for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2510_03557_b200.box import BoxGeometry
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.gravity import ForceSplit, short_range_gravity_kernel
    from paper_2510_03557_b200.ic import make_clustered_ic, make_zeldovich_ic
    from paper_2510_03557_b200.lane import EvalMode, eval_interaction_list
    from paper_2510_03557_b200.resident import ResidentRank, StepConfig
    box = BoxGeometry(1.0)
    for p in (make_zeldovich_ic(16, box, 1.0), make_clustered_ic(12, box, seed=3)):
        npd = round((p.n / 2) ** (1 / 3))
        d = 1.0 / npd
        reach = max(5 * d, 2 * float(p.smoothing.max()))
        cfg = StepConfig(box=box, bin_width=reach * (1 + 1e-9), max_leaf_size=256, r_s=d,
                         r_cut=5 * d, softening=(1.0 / p.n ** (1 / 3)) / 50)
        rr = ResidentRank(p.copy(), cfg)
        rr.step()
        rr.step(timing=True)
        print("pairs", rr.gravity_pair_count())
        q = p.copy()
        mesh = build_mesh_and_leaves(q, box, reach * (1 + 1e-9), 64)
        il = assemble_interaction_lists(mesh, reach, 0)
        gk = short_range_gravity_kernel(ForceSplit(r_s=d, r_cut=5 * d), cfg.softening)
        for mode in (EvalMode.RELAXED, EvalMode.DETERMINISTIC):
            eval_interaction_list(gk, il, q.state_matrix(5 / 3), mesh, mode=mode)
    torch.cuda.synchronize()
    print("sanitize step ok")


if __name__ == "__main__":
    main()
