#!/bin/bash
# final verification on the committed code: GPU suite, smoke, a c2 and a short c4 line
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/v_smoke.log
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v_bench_c2.log 2>&1
echo "rc=$?" >> gpurun_out/v_bench_c2.log
timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4final > gpurun_out/v_c4.log 2>&1
echo "rc=$?" >> gpurun_out/v_c4.log
