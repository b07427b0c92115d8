#!/bin/bash
# A/B of library variants on the C2 (or $CFG) step: bench.py per variant, alternated.
#   bash scripts/ab_bench.sh "name=path name2=path2" [rounds]
cd $GRAFT_REPO_ROOT
CFG=${CFG:-c2}
for r in $(seq 1 ${2:-2}); do
  for kv in $1; do
    name=${kv%%=*}; lib=${kv#*=}
    [ "$lib" = "default" ] && lib=""
    BT_LIB_PATH=$lib python bench.py --config $CFG --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_${name}_$r.json 2> gpurun_out/ab_${name}_$r.err
    python - "$name" "gpurun_out/ab_${name}_$r.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
k = d["kernels"]
print(sys.argv[1], "ms/step", d["ms_per_step"], " ".join(f"{n}={v['us']:.2f}" for n, v in k.items()))
PY
  done
done
