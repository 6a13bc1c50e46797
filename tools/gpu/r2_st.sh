#!/bin/bash
cd $GRAFT_REPO_ROOT
bash tools/gpu/r2_tq.sh stencil
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_gravity_only.py tests/test_gpu_mutation.py -x -q -p no:cacheprovider -k "not c4" >> gpurun_out/t_stencil.log 2>&1
python tools/ab_step.py --config c4 --steps 5 --tag stencil >> gpurun_out/t_stencil.log 2>&1
