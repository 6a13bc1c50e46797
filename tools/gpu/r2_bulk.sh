#!/bin/bash
# bulk-async (cp.async.bulk + mbarrier) source ring in the SPH sweeps: A/B at c2 and c4,
# then the SPH parity cases with the ring on
cd $GRAFT_REPO_ROOT
for b in 0 1 2 0 1 2; do
  HB_SPH_BULK=$b python tools/ab_step.py --config c2 --steps 10 --tag bulk$b >> gpurun_out/bulk_ab.log 2>&1
done
for b in 0 2; do
  HB_SPH_BULK=$b python tools/ab_step.py --config c4 --steps 3 --tag bulk$b >> gpurun_out/bulk_ab.log 2>&1
done
HB_SPH_BULK=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py -x -q -p no:cacheprovider -k "c1 or step or c2" > gpurun_out/bulk_parity.log 2>&1
echo "rc=$?" >> gpurun_out/bulk_parity.log
# DRAM bytes of every kernel of one c2 step (build_hbm_r02)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hbm_c2_r02.csv python tools/profile_step.py --config c2 --steps 1 > gpurun_out/hbm_c2_r02.log 2>&1
echo "rc=$?" >> gpurun_out/hbm_c2_r02.log
