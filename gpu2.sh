cd $GRAFT_REPO_ROOT
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout -s KILL 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
tail -3 gpurun_out/bench_c2.err
timeout -s KILL 600 python bench.py --config c3 --no-cpu-baseline --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
tail -3 gpurun_out/bench_c3.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 90 -c 90 --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_forward.py --config c2 --iters 2 > /dev/null 2>&1; echo "ncu rc=$?"
cat gpurun_out/bench_c2.json gpurun_out/bench_c3.json
