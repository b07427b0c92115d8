# attn-out + LN0 as the cluster kernel over 3 waves of row blocks at C3 (FFN2 unfused) vs the default
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "any_shape" > gpurun_out/any_shape_test.txt 2>&1; echo TEST_RC=$? >> gpurun_out/any_shape_test.txt
bash scripts/ab_env.sh "BT_FUSED_LN=1 BT_GEMM_LN_WAVES=3" c3
