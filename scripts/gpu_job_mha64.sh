#!/bin/bash
# Experimental four-CTAs-per-SM MHA (BT_MHA64=1): the MHA / forward GPU tests
# routed through it, then launch timing against the default kernels.
cd $GRAFT_REPO_ROOT
export BT_MHA_SEG=0 BT_MHA_LIST=0
BT_MHA64=1 timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "mha" 2>&1 | tail -3
echo "== time"
for r in 1 2; do
  echo "-- default (seg/list off)"; timeout -s KILL 200 python scripts/mha_time.py c2 c3 c5
  echo "-- mha64"; BT_MHA64=1 timeout -s KILL 200 python scripts/mha_time.py c2 c3 c5
done
unset BT_MHA_SEG BT_MHA_LIST
echo "-- default policy (seg + list)"; timeout -s KILL 200 python scripts/mha_time.py c2 c3 c5
