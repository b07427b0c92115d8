# FMA-pipe share of the FFN1 GELU (GEMM_GELU_FMA = n of every 4 pairs): numerics + C2/C3 A/B
cd $GRAFT_REPO_ROOT
for n in 1 2 3; do
 lib=abvar/gelu$n/libbt200.so
 BT_LIB_PATH=$lib timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "test_gemm and not streamk" > gpurun_out/gelu_tests_$n.txt 2>&1; echo "variant $lib tests rc=$?"; tail -1 gpurun_out/gelu_tests_$n.txt
done
BT_LIB_PATH=abvar/gelu2/libbt200.so timeout 300 python -m pytest tests/test_gpu_encoder.py -q -k "c2_vs_oracle or golden" > gpurun_out/gelu_enc.txt 2>&1; echo "enc rc=$?"; tail -1 gpurun_out/gelu_enc.txt
bash scripts/ab_bench.sh "base=default g1=abvar/gelu1/libbt200.so g2=abvar/gelu2/libbt200.so g3=abvar/gelu3/libbt200.so" 3
CFG=c3 bash scripts/ab_bench.sh "base=default g2=abvar/gelu2/libbt200.so" 2
