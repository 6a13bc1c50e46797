bash tools/gpu/nx_default.sh 4
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --config c2 > gpurun_out/final_c2_n$n.json 2> gpurun_out/final_c2_n$n.err; echo "c2 n$n rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/final_c2_n$n.json').read().strip().splitlines()[-1]);print('c2 n$n', round(d['value']/1e6,1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), 'frac', round(d['roofline']['frac'],4), d['clocks'])"
done
