cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python scripts/sweep_c4.py --out gpurun_out/c4_sweep.csv > gpurun_out/c4.log 2>&1; echo "c4 rc=$?"; tail -3 gpurun_out/c4.log
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/bench_c5.json'))
print(d['ms_per_step'], d['value'], d['tokens_per_s'], d['roofline'], d['e2e'])"
tail -2 gpurun_out/bench_c5.err
