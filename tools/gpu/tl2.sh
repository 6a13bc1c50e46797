for l in 2 0; do
  HB_GRAV_TILE_LEVELS=$l timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tl_$l.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/tl_$l.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print('levels $l', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'k_gravity', round(ph['k_gravity'],3), 'gravity phase', round(ph['gravity'],3))"
done
