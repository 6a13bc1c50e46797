#!/bin/bash
# ncu launch list (device time per kernel) of two c2 force steps and of the c4 bench step
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config c2 --steps 2"
$CMD > gpurun_out/launch_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2_r2.csv $CMD > gpurun_out/launch_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/launch_ncu.log
