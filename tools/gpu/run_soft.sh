set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_soft.json 2> gpurun_out/bench_soft.err; echo "bench rc=$?"
HB_GRAVITY_MODE=3 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_m3.json 2> gpurun_out/bench_m3.err; echo "bench m3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gravity -c 1 -f -o gpurun_out/grav_soft python tools/profile_step.py --steps 1 > gpurun_out/ncu_soft.log 2>&1; echo "ncu rc=$?"
