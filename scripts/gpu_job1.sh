cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout -s KILL 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python scripts/profile_forward.py --config c2 --iters 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 --launch-skip 0 -c 4 -o gpurun_out/c2_gemm python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:mha_fwd -c 1 -o gpurun_out/c2_mha python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_mha.log 2>&1; echo "ncu mha rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"ln_bias|pack|unpack|plan" -c 6 -o gpurun_out/c2_mem python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_mem.log 2>&1; echo "ncu mem rc=$?"
cat gpurun_out/bench_c2.json
