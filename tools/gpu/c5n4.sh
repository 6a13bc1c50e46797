timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --config c2 > gpurun_out/c2n2_chk.json 2> gpurun_out/c2n2_chk.err; echo "c2 n2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/c2n2_chk.json').read().strip().splitlines()[-1]);print('c2 n2', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1))"
( while sleep 10; do nvidia-smi --query-gpu=memory.used --format=csv,noheader | tr '\n' ' '; free -g | sed -n 2p | awk '{print $3}'; done ) > gpurun_out/c5_mem.log 2>&1 &
MON=$!
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 4 --config c5 --steps 5 --warmup 3 > gpurun_out/c5_n4.json 2> gpurun_out/c5_n4.err; echo "c5 n4 rc=$?"
kill $MON
tail -3 gpurun_out/c5_n4.err | cut -c1-300
python -c "import json;d=json.loads(open('gpurun_out/c5_n4.json').read().strip().splitlines()[-1]);print('c5 n4', round(d['value']/1e6,1), d['ms_per_step'], 'e2e', round(d['e2e']['value']/1e6,1), 'frac', round(d['roofline']['frac'],4), d['clocks'], d['phases_ms'].get('exchange'))"
sort -t' ' -k1 -n gpurun_out/c5_mem.log | tail -2
