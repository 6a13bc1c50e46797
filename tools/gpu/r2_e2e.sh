#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "host_stepper or resident" > gpurun_out/e2e_t.log 2>&1
echo "rc=$?" >> gpurun_out/e2e_t.log
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_bench.log 2>&1
echo "rc=$?" >> gpurun_out/e2e_bench.log
