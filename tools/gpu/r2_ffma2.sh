#!/bin/bash
# packed FP32x2 gravity flush: c2 / c4 step timing, gravity parity (C1, full-size sampled, DM)
cd $GRAFT_REPO_ROOT
python tools/ab_step.py --config c2 --steps 10 --tag ffma2 > gpurun_out/ffma2_ab.log 2>&1
python tools/ab_step.py --config c4 --steps 3 --tag ffma2 >> gpurun_out/ffma2_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_gravity_only.py -q -p no:cacheprovider > gpurun_out/ffma2_parity.log 2>&1
echo "rc=$?" >> gpurun_out/ffma2_parity.log
