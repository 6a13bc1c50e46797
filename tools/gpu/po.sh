timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for ov in 0 1; do
  HB_GRAV_PREP_OVERLAP=$ov timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_po$ov.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_po$ov.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print('overlap $ov', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), {k:round(v,2) for k,v in ph.items()})"
done
