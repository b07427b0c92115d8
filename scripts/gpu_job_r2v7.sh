#!/bin/bash
# Round-2 v7 profile: the round profile job, the C1 bench line, the C4 sweep
# and the GPU test suite (after the segment-kernel policy and plan changes).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.txt
bash scripts/gpu_job_profile.sh
timeout -s KILL 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?"
timeout -s KILL 1500 python scripts/sweep_c4.py --out gpurun_out/c4_sweep.csv --repeats 3 > gpurun_out/c4_sweep.log 2>&1; echo "c4 rc=$?"
tail -3 gpurun_out/c4_sweep.log
