for lv in 0 2 3; do
  HB_GRAV_TILE_LEVELS=$lv timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_tl$lv.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_tl$lv.json').read().strip().splitlines()[-1]);print('levels $lv', round(d['value']/1e6,1), 'k_gravity', round(d['phases_ms']['k_gravity'],3), 'frac', round(d['roofline']['frac'],4))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gravity -c 1 -f -o gpurun_out/grav_tl2 python tools/profile_step.py --steps 1 > gpurun_out/ncu_tl2.log 2>&1; echo "ncu rc=$?"
