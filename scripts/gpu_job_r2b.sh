#!/bin/bash
cd $GRAFT_REPO_ROOT
./scripts/micro/tmem_bw > gpurun_out/tmem_bw.txt 2>&1
./scripts/micro/mufu_bench > gpurun_out/mufu_bench.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_ladder.py -q -rf > gpurun_out/pytest_ladder.log 2>&1
BT_AUTOTUNE_VERBOSE=1 timeout 600 python scripts/gemm_probe.py c2 0 -256 -192 -128 128 192 256 > gpurun_out/gemm_probe_c2.txt 2> gpurun_out/gemm_probe_c2.err
timeout 600 python scripts/gemm_probe.py c3 0 -256 -128 256 > gpurun_out/gemm_probe_c3.txt 2>&1
