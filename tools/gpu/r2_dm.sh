#!/bin/bash
# fused tile boxes: quick parity + c2/c4 timing; DM-only 512^3 gravity: bin tiles (mode 0) vs half-warp tiles (mode 2)
cd $GRAFT_REPO_ROOT
bash tools/gpu/r2_tq.sh fusedbox
python tools/ab_step.py --config c4 --steps 5 --tag fusedbox >> gpurun_out/t_fusedbox.log 2>&1
for m in 0 2; do HB_GRAVITY_MODE=$m python tools/ab_step.py --config c5 --npd 512 --steps 5 --tag dm_mode$m; done > gpurun_out/dm_ab.log 2>&1
