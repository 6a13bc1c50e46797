#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_crk_gradients.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gradient or c1" > gpurun_out/grad.log 2>&1
echo "rc=$?" >> gpurun_out/grad.log
