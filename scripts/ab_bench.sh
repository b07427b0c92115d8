# A/B: bench the working tree against a copy of HEAD built under _ab/
# usage: bash scripts/ab_bench.sh [configs...]   (default: c2 c3)
cd $GRAFT_REPO_ROOT
CFGS=${@:-c2 c3}
for i in 1 2 3; do
 for v in new old; do
  if [ $v = new ]; then D=.; else D=_ab; fi
  for c in $CFGS; do
   (cd $D && timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], {k: round(v['us'],2) for k, v in d.get('kernels',{}).items() if k.startswith('gemm')})")
  done
 done
done
