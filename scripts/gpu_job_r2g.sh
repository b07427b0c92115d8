#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_mha2.py -x -q -rf > gpurun_out/pytest_mha2.log 2>&1
echo "mha2 rc=$?" >> gpurun_out/pytest_mha2.log
tail -4 gpurun_out/pytest_mha2.log
if grep -q " passed" gpurun_out/pytest_mha2.log && ! grep -q "failed" gpurun_out/pytest_mha2.log; then
  for cfg in c2 c3 c5; do
    st=20; [ $cfg = c5 ] && st=4
    for v in 0 1; do
      BT_MHA_V2=$v timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_mha_${cfg}_v$v.json 2> gpurun_out/ab_mha_${cfg}_v$v.err
      python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_mha_${cfg}_v$v.json').read().strip().splitlines()[-1]); print('$cfg v$v', d['ms_per_step'], 'mha', d['kernels']['mha']['us'], d['clocks'])"
    done
  done
fi
