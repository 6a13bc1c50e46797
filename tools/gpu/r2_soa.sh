#!/bin/bash
# SoA rows (no (n,12) state matrix): full GPU suite, c2 / c4 step timing, bench c4
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/soa_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/soa_pytest.log
python tools/ab_step.py --config c2 --steps 10 --tag soa > gpurun_out/soa_ab_c2.log 2>&1
python tools/ab_step.py --config c4 --steps 5 --tag soa > gpurun_out/soa_ab_c4.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/soa_bench_c4.log 2>&1
echo "rc=$?" >> gpurun_out/soa_bench_c4.log
