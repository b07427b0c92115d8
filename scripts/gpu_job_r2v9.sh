#!/bin/bash
# Round-2 v9 profile (last session): GPU suite, the round profile job (bench
# C2/C3/C5 + reference arm + ncu launch list and full captures), C1 line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.txt
bash scripts/gpu_job_profile.sh
timeout -s KILL 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?"
