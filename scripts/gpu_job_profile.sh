# Round profile: bench lines (C2 default with cpu_baseline, C3, C5), the
# reference arm, steady-state ncu launch list + full captures (C2, C3, C5).
# Outputs in gpurun_out/; copy the summaries into profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none"
timeout -s KILL 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout -s KILL 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout -s KILL 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/c2_launches_ss.csv python scripts/profile_forward.py --config c2 --iters 1 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 $P --set full --import-source on -k regex:"gemm|mha|ln_bias|forward_prologue" -c 8 -o gpurun_out/c2_all_ss python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout -s KILL 900 $P --set full -k regex:"gemm|mha|ln_bias|forward_prologue" -c 8 -o gpurun_out/c3_all_ss python scripts/profile_forward.py --config c3 --iters 1 > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout -s KILL 1200 $P --set full -k regex:"gemm|mha|ln_bias|forward_prologue" -c 8 -o gpurun_out/c5_all_ss python scripts/profile_forward.py --config c5 --iters 1 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
python scripts/ncu_summary.py gpurun_out/c2_all_ss.ncu-rep gpurun_out/c3_all_ss.ncu-rep gpurun_out/c5_all_ss.ncu-rep --out gpurun_out/ncu_summary.json --traffic gpurun_out/ncu_traffic.json > gpurun_out/ncu_summary.txt 2>&1; echo "summary rc=$?"
for c in c2 c3 c5; do ncu -i gpurun_out/${c}_all_ss.ncu-rep --page details --csv > gpurun_out/${c}_details.csv 2>/dev/null; done
mkdir -p /tmp/reps && mv gpurun_out/*.ncu-rep /tmp/reps/ 2>/dev/null; ls -la gpurun_out | head -30
