"""Timeline of one end-to-end (host-buffer) force step at c2, N = 1.

Replaces HostStepper's internal events with timing-enabled ones and prints
when each H2D group lands, when the SPH passes, the first gravity half and the
step finish, and when the call returns (all D2H drained), in ms from the call's
start.  Diagnostic only: `python tools/e2e_timeline.py [--config c2]`."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import bench
from paper_2510_03557_b200.resident import PASS_ALL, STEP_FIELDS, HostStepper


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--phases", action="store_true",
                    help="also run the step with its phase timer (the step then syncs at "
                         "its end, so the outputs' copy-out no longer overlaps gravity) and "
                         "print the phase times under the concurrent uploads")
    args = ap.parse_args()
    p, cfg, meta = bench.make_workload(args.config)
    rr = bench._make_rank(args, p, cfg, 0, 1, meta)
    pinned_in = {f: torch.from_numpy(np.ascontiguousarray(getattr(p, f))).pin_memory()
                 for f in STEP_FIELDS}
    out_names = ("grav", "hydro", "ncount", "crk_A", "crk_B", "perm")
    pinned_out = {k: torch.empty(rr.out[k].shape, dtype=rr.out[k].dtype).pin_memory()
                  for k in out_names}
    pinned_out["density"] = torch.empty(rr.n, dtype=torch.float64).pin_memory()
    hs = HostStepper(rr, pinned_in, pinned_out, PASS_ALL)
    names = ("ev_first", "ev_fields", "ev_late", "ev_last", "ev_sph", "ev_ghalf", "ev_done")
    for nm in names:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        setattr(hs, nm, ev)
    for _ in range(3):
        hs()
    torch.cuda.synchronize()
    rows = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hs()
        e1.record()
        torch.cuda.synchronize()
        rows.append([e0.elapsed_time(getattr(hs, nm)) for nm in names] + [e0.elapsed_time(e1)])
    med = np.median(np.array(rows), axis=0)
    for nm, v in zip(names + ("return",), med):
        print(f"{nm:10s} {v:8.3f} ms")
    h2d = sum(t.numel() * t.element_size() for t in pinned_in.values())
    d2h = sum(t.numel() * t.element_size() for t in pinned_out.values())
    print(f"h2d {h2d / 1e6:.1f} MB  d2h {d2h / 1e6:.1f} MB")
    groups = {"FIRST": HostStepper.FIRST, "EARLY": HostStepper.EARLY, "LATE4": HostStepper.LATE4,
              "LAST4": HostStepper.LAST4}
    print("four groups:", hs.four_groups)
    for g, fs in groups.items():
        print(g, {f: round(pinned_in[f].numel() * pinned_in[f].element_size() / 1e6, 1) for f in fs})
    print({k: round(v.numel() * v.element_size() / 1e6, 1) for k, v in pinned_out.items()})
    if args.phases:
        step0 = rr.step

        def timed(*a, **k):   # the timed step checks its own status: mark the word clean
            out = step0(*a, **{**k, "timing": True})
            hs.status[0], hs.status[1], hs.status[2] = -1, 0, 0
            return out
        rr.step = timed
        hs()
        print("phases under uploads:", {k: round(v, 3) for k, v in rr.last["ms_phase"].items()})
        rr.step = step0
        rr.step(PASS_ALL, timing=True)
        print("phases device-only:  ", {k: round(v, 3) for k, v in rr.last["ms_phase"].items()})


if __name__ == "__main__":
    main()
