"""Time the parts of one adapt_smoothing_length iteration at c2 (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import numpy as np
    import torch
    from bench import make_workload
    from paper_2510_03557_b200 import _native as N
    from paper_2510_03557_b200.cmtree import assemble_interaction_lists, build_mesh_and_leaves
    from paper_2510_03557_b200.kernels import neighbor_count_kernel
    from paper_2510_03557_b200.lane import eval_on_device
    from paper_2510_03557_b200.particles import COL_H
    p, cfg, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
    mesh = build_mesh_and_leaves(p, cfg.box, cfg.bin_width, cfg.max_leaf_size)
    il = assemble_interaction_lists(mesh, min(2 * 0.5 * cfg.bin_width, cfg.bin_width), 0)
    st = N.dev(p.state_matrix(cfg.eos_gamma), torch.float64)
    ps = N.dev(p.image_shift, torch.int8)
    la, lb, lsh = (N.dev(il.leaf_a, torch.int64), N.dev(il.leaf_b, torch.int64),
                   N.dev(il.shift, torch.int8))
    ls, le = N.dev(mesh.leaf_start, torch.int64), N.dev(mesh.leaf_end, torch.int64)
    k = neighbor_count_kernel(2 * float(p.smoothing.max()))
    T = {}

    def tm(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        T.setdefault(name, []).append((time.perf_counter() - t0) * 1e3)
        return r
    for _ in range(4):
        tm("h_column", lambda: st[:, COL_H].copy_(torch.from_numpy(p.smoothing)))
        out, _ = tm("eval", lambda: eval_on_device(k, st, ps, None, la, lb, lsh, ls, le,
                                                    mesh.n_leaves, 1.0, True, 8))
        tm("d2h", lambda: out.cpu().numpy())
    print({k: round(float(np.median(v)), 2) for k, v in T.items()}, "entries", len(il),
          "leaves", mesh.n_leaves)


if __name__ == "__main__":
    main()
