cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
 for v in "base||" "fused2|BT_FUSED_LN=2|" "fused2mc|BT_FUSED_LN=2|abv/glnmc.so"; do
  IFS='|' read name envs lib <<< "$v"
  for c in c2 c3; do
   env $envs BT_LIB_PATH=$lib timeout -s KILL 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$name $c', d['ms_per_step'], d['clocks']['sm_mhz'], {k: round(v['us'],2) for k, v in d.get('kernels',{}).items() if 'ffn2' in k or 'ln1' in k or 'ln' in k})"
  done
 done
done
