#!/bin/bash
# packed FP32x2 SPH pair bodies (HB_SPH_PACK: 1 pass B, 2 pass A): c2 / c4 timing + SPH parity
cd $GRAFT_REPO_ROOT
for p in 0 3 0 3; do
  HB_SPH_PACK=$p python tools/ab_step.py --config c2 --steps 10 --tag pack$p >> gpurun_out/pack_ab.log 2>&1
done
HB_SPH_PACK=3 python tools/ab_step.py --config c4 --steps 3 --tag pack3 >> gpurun_out/pack_ab.log 2>&1
HB_SPH_PACK=3 HB_PARITY_LOG=gpurun_out/pack_err.jsonl timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_mutation.py tests/test_gpu_crk_gradients.py -q -p no:cacheprovider > gpurun_out/pack_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pack_parity.log
