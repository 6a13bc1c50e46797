bash tools/gpu/final_r01_n4.sh
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus 4 --config c5 --steps 5 --warmup 3 > gpurun_out/final_c5_n4.json 2> gpurun_out/final_c5_n4.err; echo "c5 n4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/final_c5_n4.json').read().strip().splitlines()[-1]);print('c5 n4', round(d['value']/1e6,1), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']/1e6,1), 'frac', round(d['roofline']['frac'],4), d['clocks'])"
