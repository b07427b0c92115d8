#!/bin/bash
cd $GRAFT_REPO_ROOT
export BT_MHA_SEG=0 BT_MHA_LIST=0 BT_MHA64=1
O=gpurun_out/mha64_cases.txt; : > $O
for c in "256 2 100 150 60" "700 2 600 300 700" "256 2 100" "256 2 150" "700 2 700" "700 2 300" "700 2 600" "512 4 300 17 256" "64 1 64" "128 1 1" "200 2 129"; do
  echo "== $c" >> $O
  timeout -s KILL 40 python scripts/mha64_cases.py $c >> $O 2>&1; echo "rc=$?" >> $O
done
cat $O
