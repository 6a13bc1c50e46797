# ncu metrics of k_gravity (groups 1) vs k_gravity_g4 (groups 4)
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__average_warp_latency_issue_stalled_short_scoreboard,smsp__average_warp_latency_issue_stalled_mio_throttle,smsp__inst_executed_op_shared_ld.sum
for g in 1 4; do
  HB_GRAV_GROUPS=$g timeout 600 ncu --metrics $M --clock-control none -k regex:k_gravity -c 1 --csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_g$g.csv 2>gpurun_out/ncu_g$g.err; echo "g$g rc=$?"
done
