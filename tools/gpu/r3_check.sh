#!/bin/bash
# fresh-container re-check: GPU suite, smoke, a short default bench line
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 -p no:cacheprovider > gpurun_out/r3_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r3_smoke.log
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3_bench_c2.log 2>&1
echo "rc=$?" >> gpurun_out/r3_bench_c2.log
