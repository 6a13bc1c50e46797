# the driver's N-GPU launches with the default config, both arms: bash tools/gpu/nx_default.sh N
N=${1:-2}
( while sleep 5; do free -g | sed -n 2p | awk '{print $3}'; done ) > gpurun_out/n${N}_hostmem.log 2>&1 &
MON=$!
T0=$(date +%s)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/n${N}_ours.json 2> gpurun_out/n${N}_ours.err; echo "ours rc=$? $(( $(date +%s) - T0 )) s"
T1=$(date +%s)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus $N --steps 10 --warmup 3 > gpurun_out/n${N}_ref.json 2> gpurun_out/n${N}_ref.err; echo "ref rc=$? $(( $(date +%s) - T1 )) s"
kill $MON
echo "host mem total GB: $(free -g | sed -n 2p | awk '{print $2}'), peak used GB: $(sort -n gpurun_out/n${N}_hostmem.log | tail -1)"
python - <<PY
import json
for f in ("n${N}_ours", "n${N}_ref"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["config"].get("config"), round(d["value"] / 1e6, 2), round(d["ms_per_step"], 1), d.get("e2e", {}).get("value"), d.get("clocks", {}).get("sm_mhz"))
    except Exception as e:
        print(f, "ERR", e)
PY
