timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for c in c2 c3; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/kd_$c.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/kd_$c.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print('$c', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'build', round(ph['build'],3))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_kd_split -c 1 --csv python tools/profile_step.py --steps 1 2>/dev/null | grep k_kd_split | tail -1 | awk -F'","' '{print "k_kd_split", $(NF)}'
