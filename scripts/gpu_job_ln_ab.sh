#!/bin/bash
# LayerNorm A/B: pipelined rows (working tree) vs abv/oldln.so, C2 (+ BT_LN_SMEM_SMALL=1), C3, C5; LN tests.
cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "ln or layernorm" 2>&1 | tail -2
for r in 1 2; do
  for c in c2 c3; do
    CFG=$c bash scripts/ab_bench.sh "new=default old=abv/oldln.so" 1 2>&1 | grep -o "^[a-z]* ms/step [0-9.]*\|ln[0-9a-z_]*=[0-9.]*" | tr '\n' ' '; echo " [$c]"
  done
  BT_LN_SMEM_SMALL=1 CFG=c2 bash scripts/ab_bench.sh "new_smem=default" 1 2>&1 | grep -o "^[a-z_]* ms/step [0-9.]*\|ln[0-9a-z_]*=[0-9.]*" | tr '\n' ' '; echo " [c2 smem-small]"
done
for v in default abv/oldln.so; do
  BT_LIB_PATH=$([ $v = default ] || echo $v) timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5', d['ms_per_step'], {k: round(v['us'],1) for k,v in d['kernels'].items() if 'ln' in k}, d['clocks']['sm_mhz'])"
done
