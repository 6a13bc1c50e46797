#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_nccl.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/nccl2.log 2>&1
echo "rc=$?" >> gpurun_out/nccl2.log
