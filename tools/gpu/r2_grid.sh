#!/bin/bash
# grid-quantised segment origins (exact D) + packed SPH mask build: error statistics for
# HB_GRAV_ACC 0 / 1 / 2, c2 timing, then the full GPU suite at the default
cd $GRAFT_REPO_ROOT
for acc in 0 1 2; do
  HB_GRAV_ACC=$acc python tools/ab_step.py --config c2 --steps 10 --tag grid_acc$acc >> gpurun_out/grid_ab.log 2>&1
  HB_GRAV_ACC=$acc HB_PARITY_LOG=gpurun_out/grid_err_$acc.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -p no:cacheprovider -k "dark_matter or c3" > gpurun_out/grid_par_$acc.log 2>&1
done
HB_PARITY_LOG=gpurun_out/grid_err_all.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/grid_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/grid_pytest.log
