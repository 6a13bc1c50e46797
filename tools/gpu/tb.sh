timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_tb.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_tb.json').read().strip().splitlines()[-1]);print(round(d['value']/1e6,1), d['phases_ms'], d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01e.csv python tools/profile_step.py --steps 2 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
