#!/bin/bash
# A/B: persistent gravity grid with a tile counter (HB_GRAV_PERSIST 1) vs one tile per warp, parity with the default
cd $GRAFT_REPO_ROOT
for s in 0 1 0 1; do HB_GRAV_PERSIST=$s timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag p$s; done > gpurun_out/persist_ab.log 2>&1
for s in 0 1; do HB_GRAV_PERSIST=$s timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4p$s; done >> gpurun_out/persist_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_gravity_only.py tests/test_gpu_mutation.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/persist_parity.log 2>&1
echo "rc=$?" >> gpurun_out/persist_parity.log
