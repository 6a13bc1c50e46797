#!/bin/bash
# k_gravity at c4: DRAM bytes and executed FP32 instruction counts (few passes)
cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --config c4 --steps 2"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum
$CMD > gpurun_out/ncu_c4g_plain.log 2>&1 && \
timeout 2400 ncu --metrics $M --clock-control none -k regex:"k_gravity" -s 1 -c 1 --csv \
  --log-file gpurun_out/ncu_c4g.csv $CMD > gpurun_out/ncu_c4g.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c4g.log
CMD2="python tools/profile_step.py --config c2 --steps 2"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gravity|k_sph_force|k_sph_density" -s 3 -c 3 -o gpurun_out/prof_c2_final $CMD2 > gpurun_out/ncu_c2f.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c2f.log
