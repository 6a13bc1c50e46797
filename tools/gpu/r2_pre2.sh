#!/bin/bash
# A/B of the pre-pass-B gravity chunk in host-buffer steps (HB_GRAV_PRE)
cd $GRAFT_REPO_ROOT
for p in 0 1 0 1; do
  echo "HB_GRAV_PRE=$p" >> gpurun_out/pre2_tl.log
  HB_GRAV_PRE=$p timeout 900 python tools/e2e_timeline.py --config c4 >> gpurun_out/pre2_tl.log 2>&1
done
