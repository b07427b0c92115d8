# Round profile: bench lines (C2 default with cpu_baseline, C3, C5), the
# reference arm, steady-state ncu launch list + full captures.  Outputs in
# gpurun_out/; copy the summaries into profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none"
timeout -s KILL 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout -s KILL 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout -s KILL 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/c2_launches_ss.csv python scripts/profile_forward.py --config c2 --iters 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 $P --set full --import-source on -k regex:"gemm|mha_fwd|ln_bias|pack|unpack|plan" -c 12 -o gpurun_out/c2_all_ss python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout -s KILL 900 $P --set full -k regex:"gemm|mha_fwd|ln_bias" -c 7 -o gpurun_out/c3_all_ss python scripts/profile_forward.py --config c3 --iters 1 > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
