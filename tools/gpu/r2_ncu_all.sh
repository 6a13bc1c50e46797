#!/bin/bash
cd $GRAFT_REPO_ROOT
bash tools/gpu/r2_launch.sh
bash tools/gpu/r2_ncu_c4.sh
