# end-of-round check: GPU suite, smoke(), the C5 line (numpy-input e2e policy) and the default bench line
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_final.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.txt
timeout -s KILL 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_final.json 2> gpurun_out/bench_c5_final.err; echo "c5 rc=$?"
timeout -s KILL 600 python bench.py > gpurun_out/bench_c2_final.json 2> gpurun_out/bench_c2_final.err; echo "c2 rc=$?"
