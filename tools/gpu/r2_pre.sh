#!/bin/bash
# gravity of the first nb/8 bins before pass B in host-buffer steps: HostStepper parity,
# e2e timeline and bench at c4, c2 phases
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "host_stepper or resident" > gpurun_out/pre_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pre_pytest.log
python tools/ab_step.py --config c2 --steps 10 --tag pre > gpurun_out/pre_ab.log 2>&1
timeout 900 python tools/e2e_timeline.py --config c4 > gpurun_out/pre_e2e_tl.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pre_bench_c4.log 2>&1
echo "rc=$?" >> gpurun_out/pre_bench_c4.log
