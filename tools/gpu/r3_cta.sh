#!/bin/bash
# A/B: persistent gravity CTA shape (HB_GRAV_CTA: 0 = 2 x 16 warps, 24 = 1 x 24 warps at 80 registers, 32 = 1 x 32 warps)
cd $GRAFT_REPO_ROOT
for s in 0 24 32 0 24 32; do HB_GRAV_CTA=$s timeout 300 python tools/ab_step.py --config c2 --steps 10 --tag cta$s; done > gpurun_out/cta_ab.log 2>&1
for s in 0 24; do HB_GRAV_CTA=$s timeout 600 python tools/ab_step.py --config c4 --steps 3 --tag c4cta$s; done >> gpurun_out/cta_ab.log 2>&1
