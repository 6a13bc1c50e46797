timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ck_n1.json 2> gpurun_out/ck_n1.err; echo "n1 rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/ck_n2.json 2> gpurun_out/ck_n2.err; echo "n2 rc=$?"
python - <<'PY'
import json
for f in ("ck_n1", "ck_n2"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["config"]["config"], round(d["value"] / 1e6, 1), round(d["e2e"]["value"] / 1e6, 1), d["clocks"])
PY
