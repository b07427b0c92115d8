cd $GRAFT_REPO_ROOT
for e in 0 2; do echo "== ffn1 pair256 epi $e"; python scripts/gemm_trace.py 2458 3072 768 $e -256 | grep -E "event|finish|mainloop|epilogue per"; done
echo "== qkv PAIR1 256"; python scripts/gemm_trace.py 2458 2304 768 1 256 | grep -E "finish|mainloop|epilogue per"
echo "== ffn2 auto"; python scripts/gemm_trace.py 2458 768 3072 0 0 | grep -E "finish|mainloop|epilogue per"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/bench_c2.json'))
print(d['ms_per_step'], d['value'], {k:v['us'] for k,v in d['kernels'].items()})"
