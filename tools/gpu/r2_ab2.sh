#!/bin/bash
# A/B: gravity table JB 4 (8-warp CTAs) vs JB 5 (16-warp CTAs), c2 and c4
cd $GRAFT_REPO_ROOT
for cfg in c2 c4; do for jb in 4 5; do
  HB_GRAV_JBITS=$jb python tools/ab_step.py --config $cfg --steps 5 --tag jb$jb
done; done > gpurun_out/ab2.log 2>&1
