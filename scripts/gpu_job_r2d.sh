#!/bin/bash
cd $GRAFT_REPO_ROOT
for lib in "" scripts/ab/nbuf2.so; do
  tag=${lib:+nbuf2}; tag=${tag:-base}
  export BT_LIB_PATH=$lib
  for m in 0 8; do
    python scripts/gemm_trace.py 2458 3072 768 2 -256 $m > gpurun_out/trace_ffn1_${tag}_m$m.txt 2>&1
    python scripts/gemm_trace.py 2458 2304 768 1 192 $m > gpurun_out/trace_qkv_${tag}_m$m.txt 2>&1
    python scripts/gemm_trace.py 2458 768 3072 0 -128 $m > gpurun_out/trace_ffn2_${tag}_m$m.txt 2>&1
  done
  python scripts/gemm_probe.py c2 0 > gpurun_out/gemm_probe_c2_${tag}.txt 2>&1
done
