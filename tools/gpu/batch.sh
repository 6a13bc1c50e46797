timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for b in 1 2 4 8; do
  HB_GRAV_BATCH=$b timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gb_$b.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/gb_$b.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print('batch $b', round(d['value']/1e6,1), 'k_gravity', round(ph['k_gravity'],3), 'frac', round(d['roofline']['frac'],4))"
done
