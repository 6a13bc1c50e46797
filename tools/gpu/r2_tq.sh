#!/bin/bash
# timing at c2 + the C1 oracle parity cases (quick check of a kernel change)
cd $GRAFT_REPO_ROOT
python tools/ab_step.py --config c2 --steps 10 --tag "$1" > gpurun_out/t_$1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c1 or step" >> gpurun_out/t_$1.log 2>&1
