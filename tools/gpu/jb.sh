timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for jb in 4 5; do
  HB_GRAV_JBITS=$jb timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/ab_jb$jb.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_jb$jb.json').read().strip().splitlines()[-1]);print('jbits $jb', round(d['value']/1e6,1), d['phases_ms']['gravity'], d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gravity -c 1 -f -o gpurun_out/grav_jb4 python tools/profile_step.py --steps 1 > gpurun_out/ncu_jb4.log 2>&1; echo "ncu rc=$?"
