#!/bin/bash
# Full GPU suite + e2e host-overhead breakdown + C2 segment-MHA trace.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/check.txt
: > $O
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O
tail -3 gpurun_out/pytest_gpu.txt >> $O
timeout -s KILL 300 python scripts/e2e_breakdown.py >> $O 2>&1
BT_LIB_PATH=abv/trace.so timeout -s KILL 300 python scripts/mha_trace.py c2 seg >> $O 2>&1
cat $O
