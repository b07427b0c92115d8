#!/bin/bash
# ncu --set full (with source) of one MHA launch at C3 and C2 and of the C2
# forward prologue; per-source-line stall CSVs for reading here.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none --set full --import-source on"
timeout -s KILL 600 $P -k regex:mha_fwd -s 2 -c 1 -o gpurun_out/mha_c3 python scripts/profile_forward.py --config c3 --iters 1 > gpurun_out/ncu_mha_c3.log 2>&1; echo "c3 rc=$?"
timeout -s KILL 600 $P -k regex:"mha_fwd|forward_prologue" -c 3 -o gpurun_out/mha_c2 python scripts/profile_forward.py --config c2 --iters 1 > gpurun_out/ncu_mha_c2.log 2>&1; echo "c2 rc=$?"
for r in mha_c3 mha_c2; do
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source cuda > gpurun_out/${r}_cuda.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out
