#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_timeline.py --config c4 > gpurun_out/e2e_tl_c4.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_bench2.log 2>&1
echo "rc=$?" >> gpurun_out/e2e_bench2.log
