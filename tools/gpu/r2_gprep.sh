#!/bin/bash
cd $GRAFT_REPO_ROOT
bash tools/gpu/r2_tq.sh gprep
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_mutation.py -x -q -p no:cacheprovider -k "c2 or mutat or clustered or dark" >> gpurun_out/t_gprep.log 2>&1
timeout 1200 python tools/e2e_timeline.py --config c4 > gpurun_out/e2e_tl_c4_gprep.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gprep_bench.log 2>&1
