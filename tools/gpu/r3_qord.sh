#!/bin/bash
# A/B: gravity table gather with one zero-row word for out-of-range lanes, tile order (HB_GRAV_QORD=0)
# vs targets in spatial quarters (1); baseline k_gravity 9.03 ms at c2; then parity with the default
cd $GRAFT_REPO_ROOT
for s in 0 1 2 0 1 2; do HB_GRAV_QORD=$s timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag q$s; done > gpurun_out/qord_ab.log 2>&1
for s in 0 2; do HB_GRAV_QORD=$s timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4q$s; done >> gpurun_out/qord_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_gravity_only.py tests/test_gpu_mutation.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/qord_parity.log 2>&1
echo "rc=$?" >> gpurun_out/qord_parity.log
CMD="python tools/profile_step.py --config c2 --steps 2"
for s in 0 1 2; do
HB_GRAV_QORD=$s timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed.sum -k regex:k_gravity -s 1 -c 1 --csv $CMD > gpurun_out/qord_ncu$s.csv 2>&1
done
