cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none"
timeout -s KILL 600 $P --set full --import-source on -k regex:gemm_bf16 -c 4 -o gpurun_out/c2_gemm_ss python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout -s KILL 600 $P --set full --import-source on -k regex:"mha_fwd|ln_bias|pack|unpack|plan" -c 7 -o gpurun_out/c2_other_ss python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_other.log 2>&1; echo "ncu other rc=$?"
timeout -s KILL 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/c2_launches_ss.csv python scripts/profile_forward.py --config c2 --iters 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 600 $P --set full -k regex:gemm_bf16 -c 4 -o gpurun_out/c3_gemm_ss python scripts/profile_forward.py --config c3 --iters 1 > gpurun_out/ncu_gemm3.log 2>&1; echo "ncu gemm c3 rc=$?"
for shp in "2458 2304 768 1 0" "2458 768 768 0 0" "2458 3072 768 2 0" "2458 768 3072 0 0"; do
  timeout -s KILL 120 python scripts/gemm_trace.py $shp > gpurun_out/trace_$(echo $shp | tr ' ' _).txt 2>&1
done
timeout -s KILL 120 python scripts/mha_trace.py c2 > gpurun_out/mha_trace_c2.txt 2>&1
timeout -s KILL 120 python scripts/mha_trace.py c3 > gpurun_out/mha_trace_c3.txt 2>&1
echo done
