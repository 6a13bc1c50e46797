#!/bin/bash
# configs[4]: gravity-only 1024^3 dark matter at 4 GPUs (+ its reference arm)
cd $GRAFT_REPO_ROOT
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 4 --config c5 --steps 5 --warmup 3 > gpurun_out/c5_n4.log 2>&1
echo "rc=$?" >> gpurun_out/c5_n4.log
timeout 1200 python bench.py --impl reference --config c5 --steps 5 --warmup 1 > gpurun_out/c5_ref.log 2>&1
echo "rc=$?" >> gpurun_out/c5_ref.log
