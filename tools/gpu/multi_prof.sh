bash tools/gpu/multi.sh ${1:-4} ${2:-c2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${1:-4} --master-addr 127.0.0.1 --master-port 29513 tools/profile_exchange_fine.py ${2:-c2} 2>&1 | grep -v OMP | tail -1
