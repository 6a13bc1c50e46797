#!/bin/bash
# validation of the current build: GPU suite (with error statistics), c2 / c4 phases,
# default bench line, e2e timeline at c4
cd $GRAFT_REPO_ROOT
HB_PARITY_LOG=gpurun_out/val_err.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/val_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/val_pytest.log
python tools/ab_step.py --config c2 --steps 10 --tag val > gpurun_out/val_ab.log 2>&1
python tools/ab_step.py --config c4 --steps 3 --tag val >> gpurun_out/val_ab.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/val_bench_c4.log 2>&1
echo "rc=$?" >> gpurun_out/val_bench_c4.log
timeout 900 python tools/e2e_timeline.py --config c4 > gpurun_out/val_e2e_tl.log 2>&1
