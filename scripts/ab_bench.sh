cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
 for v in new old; do
  if [ $v = new ]; then D=.; else D=_ab; fi
  (cd $D && timeout -s KILL 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c2', d['ms_per_step'], d['e2e']['value'])")
  (cd $D && timeout -s KILL 300 python bench.py --config c3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c3', d['ms_per_step'], [ (k['name'],round(k['us'],1)) for k in d.get('kernels',[])][:8])")
 done
done
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -k "gemm" 2>&1 | tail -3
