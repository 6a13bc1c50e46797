timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/quick.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print(round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), {k:round(v,3) for k,v in ph.items()})"
