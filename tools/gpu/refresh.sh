timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config c4 --steps 5 --warmup 3 > gpurun_out/fb_c4_n2.json 2> gpurun_out/fb_c4_n2.err; echo "c4 n2 rc=$?"
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/fb_c3_n1.json 2> gpurun_out/fb_c3_n1.err; echo "c3 n1 rc=$?"
for f in fb_c4_n2 fb_c3_n1; do
  python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01f.csv python tools/profile_step.py --steps 2 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gravity|k_sph_density|k_sph_force|k_tile_build_warp|k_kd_split|k_crk_solve" -c 7 -f -o gpurun_out/kernels_r01f python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
