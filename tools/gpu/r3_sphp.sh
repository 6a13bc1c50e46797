#!/bin/bash
# A/B: persistent SPH grids (HB_SPH_PERSIST 1) vs one tile per warp, with the persistent gravity grid; parity with the default
cd $GRAFT_REPO_ROOT
for s in 0 1 0 1; do HB_SPH_PERSIST=$s timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag sp$s; done > gpurun_out/sphp_ab.log 2>&1
for s in 0 1; do HB_SPH_PERSIST=$s timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4sp$s; done >> gpurun_out/sphp_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_crk_gradients.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py tests/test_gpu_mutation.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider > gpurun_out/sphp_parity.log 2>&1
echo "rc=$?" >> gpurun_out/sphp_parity.log
