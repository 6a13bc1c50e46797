#!/bin/bash
# k_gravity at c4: DRAM bytes and executed FP32 instruction counts, packed FP32x2 included
# (few passes; a --set full capture at c4 does not collect: ncu backs up ~160 GB per replay)
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config ${1:-c4} --steps 2"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum
for k in fadd fmul ffma fadd2 fmul2 ffma2; do M=$M,sm__sass_thread_inst_executed_op_${k}_pred_on.sum; done
$CMD > gpurun_out/ncu_g_plain.log 2>&1 && \
timeout 2400 ncu --metrics $M --clock-control none -k regex:"k_gravity" -s 1 -c 1 --csv \
  --log-file gpurun_out/ncu_${1:-c4}g.csv $CMD > gpurun_out/ncu_g.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_g.log
