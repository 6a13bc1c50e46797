# round-end refresh on one GPU (results under gpurun_out/final_*)
S() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], d.get('config',{}).get('config'), round(d['value']/1e6,3), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,3), 'frac', (d.get('roofline') or {}).get('frac'), 'clk', d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))" $1; }
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo "c2 rc=$?"; S gpurun_out/final_c2.json
timeout 900 python bench.py --impl reference > gpurun_out/final_c2_ref.json 2> gpurun_out/final_c2_ref.err; echo "ref rc=$?"; S gpurun_out/final_c2_ref.json
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo "c3 rc=$?"; S gpurun_out/final_c3.json
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4_n1.json 2> gpurun_out/final_c4_n1.err; echo "c4 rc=$?"; S gpurun_out/final_c4_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gravity|k_sph_density|k_sph_force|k_tile_build_warp|k_gather_state|k_crk_solve" -c 7 -f -o gpurun_out/final_kernels python tools/profile_step.py --steps 1 > gpurun_out/final_kernels.log 2>&1; echo "full rc=$?"
timeout 1500 python tools/bench_next.py > gpurun_out/final_next.jsonl 2> gpurun_out/final_next.err; echo "next rc=$?"; cut -c1-200 gpurun_out/final_next.jsonl
