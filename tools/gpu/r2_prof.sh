#!/bin/bash
# ncu --set full (with source) of the step's interaction kernels at c2
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config c2 --steps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gravity|k_sph_force|k_sph_density" -s 3 -c 3 \
  -o gpurun_out/prof_r2 $CMD > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu.log
