#!/bin/bash
# gravity accumulation variants (HB_GRAV_ACC): c2 timing + DM / full-size parity error statistics
cd $GRAFT_REPO_ROOT
for acc in 0 1 2 3; do
  HB_GRAV_ACC=$acc python tools/ab_step.py --config c2 --steps 10 --tag acc$acc >> gpurun_out/acc_ab.log 2>&1
  HB_GRAV_ACC=$acc HB_PARITY_LOG=gpurun_out/acc_err_$acc.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -p no:cacheprovider -k "dark_matter or c3" > gpurun_out/acc_par_$acc.log 2>&1
done
HB_GRAV_ACC=1 python tools/ab_step.py --config c4 --steps 3 --tag acc1 >> gpurun_out/acc_ab.log 2>&1
HB_GRAV_ACC=3 python tools/ab_step.py --config c4 --steps 3 --tag acc3 >> gpurun_out/acc_ab.log 2>&1
