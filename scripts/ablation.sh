# In-graph cost of each per-layer launch by difference (BT_DEBUG_SKIP):
#   bash scripts/ablation.sh [config]
cd $GRAFT_REPO_ROOT
C=${1:-c2}
for skip in "" q m a f s l; do
  BT_DEBUG_SKIP=$skip timeout -s KILL 300 python bench.py --config $C --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('skip=[$skip]', d['ms_per_step'])"
done
