# the driver's N=2 launches, default config (c4 at N > 1), both arms
T0=$(date +%s)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/n2_ours.json 2> gpurun_out/n2_ours.err; echo "ours rc=$? $(( $(date +%s) - T0 )) s"
T1=$(date +%s)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 10 --warmup 3 > gpurun_out/n2_ref.json 2> gpurun_out/n2_ref.err; echo "ref rc=$? $(( $(date +%s) - T1 )) s"
free -g | sed -n 2p
python - <<'PY'
import json
for f in ("n2_ours", "n2_ref"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["config"].get("config"), round(d["value"] / 1e6, 2), d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("cpu_baseline", {}).get("sample", "")[:160])
    except Exception as e:
        print(f, "ERR", e)
PY
