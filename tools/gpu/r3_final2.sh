#!/bin/bash
# evidence on the final kernels (persistent gravity grid): GPU suite + smoke, the default
# c4 line and its reference arm, c2 / c3 / c3k lines, the c4 launch list, k_gravity's c4
# DRAM / executed-FP32 counters, and the ncu --set full capture at c2
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=40 -p no:cacheprovider > gpurun_out/g_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/g_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench_c4.log 2>&1
echo "rc=$?" >> gpurun_out/g_bench_c4.log
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g_ref_c4.log 2>&1
echo "rc=$?" >> gpurun_out/g_ref_c4.log
for c in c2 c3 c3k; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/g_bench_$c.log
done
bash tools/gpu/r2_launch_c4.sh
bash tools/gpu/r2_ncu_c4g.sh c4
bash tools/gpu/r2_prof.sh r3
