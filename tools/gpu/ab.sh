# A/B gravity variants on c2 (bench gravity phase)
for cfg in "0 1" "0 0" "3 1" "3 0"; do
  set -- $cfg
  HB_GRAVITY_MODE=$1 HB_GRAV_PERSIST=$2 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/ab_$1_$2.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_$1_$2.json').read().strip().splitlines()[-1]);print('mode $1 persist $2', round(d['value']/1e6,1), d['phase_ms']['gravity'] if 'phase_ms' in d else d['phases_ms']['gravity'])"
done
