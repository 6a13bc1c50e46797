timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for c in 1 8; do
  HB_GRAV_TABLE_COPIES=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tc_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/tc_$c.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print('copies $c', round(d['value']/1e6,1), 'k_gravity', round(ph['k_gravity'],3), 'frac', round(d['roofline']['frac'],4))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_gravity -c 1 --csv python tools/profile_step.py --steps 1 > gpurun_out/tc_ncu.csv 2>/dev/null; echo "ncu rc=$?"
