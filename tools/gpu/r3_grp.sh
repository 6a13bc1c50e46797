#!/bin/bash
# A/B: grouped-target gravity (HB_GRAV_GROUPS 1 = one list, 2 / 4 / 8 groups) at c2 and c4, parity with the default
cd $GRAFT_REPO_ROOT
for g in 1 4 2 8; do HB_GRAV_GROUPS=$g timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag g$g; done > gpurun_out/grp_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_gravity_only.py -q -x -p no:cacheprovider > gpurun_out/grp_parity.log 2>&1
echo "rc=$?" >> gpurun_out/grp_parity.log
for g in 1 4; do HB_GRAV_GROUPS=$g timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4g$g; done >> gpurun_out/grp_ab.log 2>&1
