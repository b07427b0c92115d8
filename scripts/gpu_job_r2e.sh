#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_determinism.py -q -rf -k "gemm" > gpurun_out/pytest_gemm.log 2>&1
tail -3 gpurun_out/pytest_gemm.log
for v in old=scripts/ab/old.so new=default f32tanh=scripts/ab/f32tanh.so; do
  name=${v%%=*}; lib=${v#*=}; [ "$lib" = "default" ] && lib=""
  BT_LIB_PATH=$lib python scripts/gemm_probe.py c2 0 > gpurun_out/probe_${name}.txt 2>&1
  cat gpurun_out/probe_${name}.txt | sed "s/^/$name /" | cut -c1-120
done
bash scripts/ab_bench.sh "old=scripts/ab/old.so new=default f32tanh=scripts/ab/f32tanh.so" 2
