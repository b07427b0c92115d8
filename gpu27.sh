cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"; grep e2e gpurun_out/bench_c2.err
