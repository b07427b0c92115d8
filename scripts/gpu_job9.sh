cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k mha 2>&1 | tail -2
for P in 6 8; do
  sed -i "s/^#define BT_MHA_POLY [0-9]*/#define BT_MHA_POLY $P/" paper_2210_03052_b200/csrc/mha_sm100.cu
  python -m paper_2210_03052_b200.build > /dev/null 2>&1 || echo build failed
  echo "== POLY $P"
  for c in c2 c3; do python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c step', d['ms_per_step'], 'mha', d['kernels']['mha']['us'], d['kernels']['mha']['frac'])"; done
done
