#!/bin/bash
# round-2 final evidence: full GPU suite + smoke (as the driver runs them), the
# default bench line (K = 20, W = 5) and its reference arm, c2 / c3 / c3k lines
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=40 -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench_c4.log 2>&1
echo "rc=$?" >> gpurun_out/final_bench_c4.log
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref_c4.log 2>&1
echo "rc=$?" >> gpurun_out/final_ref_c4.log
for c in c2 c3 c3k; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/final_bench_$c.log
done
