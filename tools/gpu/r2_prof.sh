#!/bin/bash
# ncu --set full (with source) of the step's interaction kernels at c2, plus the packed
# FP32x2 instruction counters (not in the full set)
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config c2 --steps 2"
X=""
for k in fadd2 fmul2 ffma2; do X=$X${X:+,}sm__sass_thread_inst_executed_op_${k}_pred_on.sum; done
$CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --metrics $X --clock-control none --import-source on \
  -k regex:"k_gravity|k_sph_force|k_sph_density" -s 3 -c 3 \
  -o gpurun_out/prof_${1:-r2} $CMD > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu.log
