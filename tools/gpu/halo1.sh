timeout 600 python tools/debug/halo_pack_1gpu.py c4 4 5 2>&1 | tail -5
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_halo|scan|k_flags" --csv python tools/debug/halo_pack_1gpu.py c4 4 2 > gpurun_out/halo1_ncu.csv 2> gpurun_out/halo1_ncu.err; echo "ncu rc=$?"
