#!/bin/bash
# timing of the current build at c2 (+ optional ncu of the SPH kernels)
cd $GRAFT_REPO_ROOT
python tools/ab_step.py --config c2 --steps 10 --tag "$1" > gpurun_out/t_$1.log 2>&1
if [ "$2" = "prof" ]; then
  CMD="python tools/profile_step.py --config c2 --steps 2"
  $CMD > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_sph_force|k_sph_density" -s 2 -c 2 -o gpurun_out/prof_$1 $CMD > gpurun_out/prof_$1.log 2>&1
fi
