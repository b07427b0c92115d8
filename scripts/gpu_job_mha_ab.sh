#!/bin/bash
# MHA A/B: launch timing (scripts/mha_time.py) and per-block traces
# (scripts/mha_trace.py) of abv/base*.so against the working tree, plus the
# MHA GPU tests on the working tree.  Outputs in gpurun_out/mha_ab.txt.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/mha_ab.txt
: > $O
for r in 1 2; do
  for v in base new; do
    L=abv/base.so; [ $v = new ] && L=""
    echo "== $v time r$r" >> $O
    BT_LIB_PATH=$L timeout -s KILL 300 python scripts/mha_time.py c2 c3 c5 >> $O 2>&1
  done
done
for v in base new; do
  for c in c2 c3; do
    echo "== $v trace $c" >> $O
    BT_LIB_PATH=abv/${v}_trace.so timeout -s KILL 300 python scripts/mha_trace.py $c >> $O 2>&1
  done
done
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_encoder.py -x -q -m gpu -k "mha or forward" >> $O 2>&1
echo "tests rc=$?" >> $O
cat $O
