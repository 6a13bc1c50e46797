#!/bin/bash
# multi-GPU evidence on the final kernels (gpurun --gpus 4): NCCL tests, c4 at N = 2 and 4, c5 at N = 4
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/m_smi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_nccl.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/m_nccl.log 2>&1
echo "rc=$?" >> gpurun_out/m_nccl.log
for N in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/m_c4_n$N.log 2>&1
  echo "rc=$?" >> gpurun_out/m_c4_n$N.log
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 4 --config c5 --steps 5 --warmup 3 > gpurun_out/m_c5_n4.log 2>&1
echo "rc=$?" >> gpurun_out/m_c5_n4.log
