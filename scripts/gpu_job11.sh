cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_encoder.py -x -q -k "layernorm or ln or encoder" 2>&1 | tail -2
for c in c2 c3; do python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c step', d['ms_per_step'], {k: (v['us'], v['frac']) for k, v in d['kernels'].items() if k.startswith('ln')})"; done
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 step', d['ms_per_step'], {k: (v['us'], v['frac']) for k, v in d['kernels'].items() if k.startswith('ln')}, d['clocks'])"
