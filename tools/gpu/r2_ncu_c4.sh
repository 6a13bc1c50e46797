#!/bin/bash
# ncu --set full of the c4 interaction kernels (one launch each, second step)
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config c4 --steps 2"
$CMD > gpurun_out/ncu_c4_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gravity|k_sph_force|k_sph_density" -s 3 -c 3 \
  -o gpurun_out/prof_c4_r2 $CMD > gpurun_out/ncu_c4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c4.log
