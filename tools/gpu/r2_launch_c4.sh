#!/bin/bash
# ncu launch list (device time per kernel) of two c4 force steps
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config c4 --steps 2"
$CMD > gpurun_out/launch_c4_plain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4_r2.csv $CMD > gpurun_out/launch_c4_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/launch_c4_ncu.log
