# usage: bash tools/gpu/multi.sh N [config]  -- GPU tests (rank 0 box) + torchrun bench at N
N=${1:-4}; CFG=${2:-c2}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for n in 1 $N; do
  if [ $n = 1 ]; then
    timeout 600 python bench.py --steps 10 --warmup 3 --config $CFG --no-cpu-baseline > gpurun_out/bench_${CFG}_n1.json 2>gpurun_out/bench_${CFG}_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 10 --warmup 3 --config $CFG > gpurun_out/bench_${CFG}_n$n.json 2>gpurun_out/bench_${CFG}_n$n.err
  fi
  python -c "import json;d=json.loads(open('gpurun_out/bench_${CFG}_n$n.json').read().strip().splitlines()[-1]);ph=d['phases_ms'];print('N=$n', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), {k:round(v,2) for k,v in ph.items()})"
done
