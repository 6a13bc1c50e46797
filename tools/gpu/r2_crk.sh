#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py -x -q -p no:cacheprovider -k "c1 or step or c2" > gpurun_out/crk.log 2>&1
echo "rc=$?" >> gpurun_out/crk.log
for cfg in c2 c4; do python tools/ab_step.py --config $cfg --steps 5 --tag crkf; done >> gpurun_out/crk.log 2>&1
