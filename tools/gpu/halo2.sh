timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python tools/debug/halo_pack_1gpu.py c4 4 5 2>&1 | tail -3
