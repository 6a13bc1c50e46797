#!/bin/bash
# exchange breakdown at c4 (host ms, device drain ms per piece) at 4 and 2 ranks
cd $GRAFT_REPO_ROOT
for N in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $((29600 + N)) tools/profile_exchange_fine.py c4 > gpurun_out/exch_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/exch_n$N.log
done
