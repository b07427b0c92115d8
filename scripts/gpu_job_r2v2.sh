#!/bin/bash
# Round-2 v2 profile: the round profile job plus the C4 sweep.
cd $GRAFT_REPO_ROOT
bash scripts/gpu_job_profile.sh
timeout -s KILL 1500 python scripts/sweep_c4.py --out gpurun_out/c4_sweep.csv --repeats 3 > gpurun_out/c4_sweep.log 2>&1; echo "c4 rc=$?"
tail -3 gpurun_out/c4_sweep.log
