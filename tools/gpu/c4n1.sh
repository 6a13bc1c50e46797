free -g | head -2; nproc; nvidia-smi --query-gpu=memory.total --format=csv,noheader; date +%s
( while sleep 20; do nvidia-smi --query-gpu=memory.used --format=csv,noheader; free -g | sed -n 2p; done ) > gpurun_out/c4_mem.log 2>&1 &
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err; echo "rc=$?"
tail -3 gpurun_out/c4_n1.err | cut -c1-300
python -c "import json;d=json.loads(open('gpurun_out/c4_n1.json').read().strip().splitlines()[-1]);print(round(d['value']/1e6,1), d['ms_per_step'], d.get('e2e',{}).get('value'), d['roofline']['frac'])"
