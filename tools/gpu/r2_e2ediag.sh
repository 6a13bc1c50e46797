#!/bin/bash
# e2e diagnostics at c4: timeline and the step's phase times while the uploads run
cd $GRAFT_REPO_ROOT
timeout 1200 python tools/e2e_timeline.py --config c4 --reps 2 --phases > gpurun_out/e2ediag_c4.log 2>&1
echo "rc=$?" >> gpurun_out/e2ediag_c4.log
