#!/bin/bash
# A/B: gravity stage layout (HB_GRAV_SOA 0 = float4 stage, 1 = blocked SoA with FADD2 / FMUL2), parity with the default
cd $GRAFT_REPO_ROOT
for s in 0 1 0 1; do HB_GRAV_SOA=$s timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag soa$s; done > gpurun_out/soa_ab.log 2>&1
for s in 0 1; do HB_GRAV_SOA=$s timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4soa$s; done >> gpurun_out/soa_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_gravity_only.py tests/test_gpu_mutation.py -q -x -p no:cacheprovider > gpurun_out/soa_parity.log 2>&1
echo "rc=$?" >> gpurun_out/soa_parity.log
