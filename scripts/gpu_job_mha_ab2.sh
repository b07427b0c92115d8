#!/bin/bash
# MHA A/B over library variants: NAME=path pairs in $VARIANTS (default: base vs working tree vs poly variants)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/mha_ab2.txt
: > $O
V=${VARIANTS:-"base=abv/base.so new= poly0=abv/poly0.so poly4=abv/poly4.so"}
for r in 1 2; do
  for kv in $V; do
    n=${kv%%=*}; L=${kv#*=}
    echo "== $n r$r" >> $O
    BT_LIB_PATH=$L timeout -s KILL 300 python scripts/mha_time.py c2 c3 c5 >> $O 2>&1
  done
done
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "mha" >> $O 2>&1
echo "tests rc=$?" >> $O
cat $O
