# headline numbers: c2 N=1 (full, with CPU baseline), c2 N=2 / N=4, c4 N=4
timeout 900 python bench.py > gpurun_out/fb_c2_n1.json 2> gpurun_out/fb_c2_n1.err; echo "c2 n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n > gpurun_out/fb_c2_n$n.json 2> gpurun_out/fb_c2_n$n.err; echo "c2 n$n rc=$?"
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29530 bench.py --gpus 4 --config c4 --steps 5 --warmup 3 > gpurun_out/fb_c4_n4.json 2> gpurun_out/fb_c4_n4.err; echo "c4 n4 rc=$?"
for f in fb_c2_n1 fb_c2_n2 fb_c2_n4 fb_c4_n4; do
  python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e6,1), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
