#!/bin/bash
# c3 (2x256^3 sigma_psi 2d) and c3k (2x128^3 clustered generator) GPU lines
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c3.log 2>&1
echo "rc=$?" >> gpurun_out/c3.log
timeout 900 python bench.py --config c3k --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c3k.log 2>&1
echo "rc=$?" >> gpurun_out/c3k.log
