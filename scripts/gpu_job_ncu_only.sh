#!/bin/bash
# ncu --set full of one layer's kernels at C2 / C3 / C5 (no bench runs), summarised.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none"
for c in c2 c3 c5; do
  timeout -s KILL 1200 $P --set full -k regex:"gemm|mha|ln_bias|forward_prologue" -c 8 -o gpurun_out/${c}_all_ss python scripts/profile_forward.py --config $c --iters 1 > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
python scripts/ncu_summary.py gpurun_out/c2_all_ss.ncu-rep gpurun_out/c3_all_ss.ncu-rep gpurun_out/c5_all_ss.ncu-rep --out gpurun_out/ncu_summary.json --traffic gpurun_out/ncu_traffic.json > gpurun_out/ncu_summary.txt 2>&1; echo "summary rc=$?"
mkdir -p /tmp/reps && mv gpurun_out/*.ncu-rep /tmp/reps/ 2>/dev/null
