# A/B one environment switch on the working tree:
#   bash scripts/ab_env.sh "BT_MHA_LIST=0" c2 c3
cd $GRAFT_REPO_ROOT
ENVB=$1; shift
CFGS=${@:-c2 c3}
for i in 1 2 3; do
 for v in A B; do
  for c in $CFGS; do
   if [ $v = A ]; then E=""; else E="$ENVB"; fi
   env $E timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v[$E] $c', d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], {k: round(v['us'],2) for k, v in d.get('kernels',{}).items() if k in ('mha',)})"
  done
 done
done
