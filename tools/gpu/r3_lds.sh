#!/bin/bash
# microbenchmark: shared-memory wavefronts of a predicated 16-B gather by active-lane pattern
cd $GRAFT_REPO_ROOT
./tools/lds_quarter > gpurun_out/lds_quarter.log 2>&1
timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum --csv ./tools/lds_quarter > gpurun_out/lds_quarter_ncu.csv 2>&1
