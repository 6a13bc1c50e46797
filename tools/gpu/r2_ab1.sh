#!/bin/bash
# A/B: gravity table resolution (JB 4 vs 5) at c2, then the DM parity test with JB 5
cd $GRAFT_REPO_ROOT
for jb in 4 5; do HB_GRAV_JBITS=$jb python tools/ab_step.py --config c2 --steps 10 --tag jb$jb; done > gpurun_out/ab1.log 2>&1
HB_GRAV_JBITS=5 timeout 600 python -m pytest tests/test_gpu_fullsize_parity.py -q -x -k dark -p no:cacheprovider >> gpurun_out/ab1.log 2>&1
bash tools/gpu/r2_prof.sh
