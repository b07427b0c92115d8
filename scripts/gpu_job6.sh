cd $GRAFT_REPO_ROOT
for P in 0 6 10 16; do
  sed -i "s/^#define BT_MHA_POLY [0-9]*/#define BT_MHA_POLY $P/" paper_2210_03052_b200/csrc/mha_sm100.cu
  python -m paper_2210_03052_b200.build > /dev/null 2>&1 || echo build failed
  echo "== POLY $P"; python scripts/mha_trace.py c2 | grep -E "item|softmax per"; python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', d['ms_per_step'], 'mha', d['kernels']['mha']['us'])"
done
