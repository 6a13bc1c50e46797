#!/bin/bash
# compute-sanitizer, one tool per call: bash tools/gpu/r2_sanitize.sh memcheck|racecheck
cd $GRAFT_REPO_ROOT
python tools/sanitize_step.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $1 --print-limit 50 python tools/sanitize_step.py > gpurun_out/san_$1.log 2>&1
echo "rc=$?" >> gpurun_out/san_$1.log
