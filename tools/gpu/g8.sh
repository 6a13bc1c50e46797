timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for m in 5 4; do
  HB_GRAVITY_MODE=$m timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/ab_m$m.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_m$m.json').read().strip().splitlines()[-1]);print('mode $m', round(d['value']/1e6,1), d['phases_ms']['gravity'], d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gravity_g8 -c 1 -f -o gpurun_out/grav_g8 python tools/profile_step.py --steps 1 > gpurun_out/ncu_g8.log 2>&1; echo "ncu rc=$?"
