#!/bin/bash
# A/B: SPH pass A residency (HB_SPH_OCC=1: 224-source stages at 8 CTAs / SM vs 256 at 7)
cd $GRAFT_REPO_ROOT
for s in 0 1 0 1; do HB_SPH_OCC=$s timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag so$s; done > gpurun_out/sphocc_ab.log 2>&1
for s in 0 1; do HB_SPH_OCC=$s timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4so$s; done >> gpurun_out/sphocc_ab.log 2>&1
HB_SPH_OCC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/sphocc_parity.log 2>&1
echo "rc=$?" >> gpurun_out/sphocc_parity.log
