#!/bin/bash
# e2e host-I/O pipeline sweep (C2, C3) + MUFU micro-benchmark + the e2e/service GPU tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/e2e.txt
: > $O
./scripts/micro/mufu_bench >> $O 2>&1
timeout -s KILL 400 python scripts/e2e_chunks.py c2 >> $O 2>&1
timeout -s KILL 400 python scripts/e2e_chunks.py c3 1 2 3 0.2,0.6,0.2 >> $O 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_encoder.py tests/test_service.py -x -q -m gpu >> $O 2>&1
echo "tests rc=$?" >> $O
cat $O
