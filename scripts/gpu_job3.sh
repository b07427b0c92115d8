cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -x -q -k mha > gpurun_out/pytest_mha.log 2>&1; echo "mha tests rc=$?"; tail -5 gpurun_out/pytest_mha.log
timeout -s KILL 120 python scripts/mha_trace.py c2 > gpurun_out/mha_trace_c2.txt 2>&1; tail -5 gpurun_out/mha_trace_c2.txt
timeout -s KILL 120 python scripts/mha_trace.py c3 > gpurun_out/mha_trace_c3.txt 2>&1; tail -5 gpurun_out/mha_trace_c3.txt
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout -s KILL 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
python - <<'PY'
import json
for c in ("c2","c3"):
    try:
        d=json.load(open(f"gpurun_out/bench_{c}.json"))
        print(c, d["ms_per_step"], d["value"], {k:v["us"] for k,v in d["kernels"].items()}, d["e2e"]["ms_per_step"])
    except Exception as e: print(c, "ERR", e)
PY
