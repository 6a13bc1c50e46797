#!/bin/bash
# pass-B lean records: parity (C1 oracle, full-size c2/c3, mutation) + timings
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_mutation.py -x -q -p no:cacheprovider -k "not c4_step" > gpurun_out/sphb_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/sphb_pytest.log
for cfg in c2 c4; do python tools/ab_step.py --config $cfg --steps 5 --tag sphb; done > gpurun_out/sphb_ab.log 2>&1
