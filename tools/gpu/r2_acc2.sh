#!/bin/bash
# gravity accumulation variants, round 2 (HB_GRAV_ACC 1 / 5 / 6 / 2): c2 timing + DM / c3 error statistics
cd $GRAFT_REPO_ROOT
for acc in 5 6 1 2; do
  HB_GRAV_ACC=$acc python tools/ab_step.py --config c2 --steps 10 --tag acc$acc >> gpurun_out/acc2_ab.log 2>&1
  HB_GRAV_ACC=$acc HB_PARITY_LOG=gpurun_out/acc2_err_$acc.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -p no:cacheprovider -k "dark_matter or c3" > gpurun_out/acc2_par_$acc.log 2>&1
done
