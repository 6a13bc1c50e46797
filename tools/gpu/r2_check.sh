#!/bin/bash
# round-2 GPU check: tests, smoke, default bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 -p no:cacheprovider > gpurun_out/r1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r1_bench.log
