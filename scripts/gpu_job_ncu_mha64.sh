#!/bin/bash
# ncu --set full with source of one four-CTA MHA launch (C3 grid mode and C5
# persistent), SASS-level stall CSVs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none --set full --import-source on"
timeout -s KILL 600 $P -k regex:mha64 -s 2 -c 1 -o gpurun_out/m64_c3 python scripts/profile_forward.py --config c3 --iters 1 > /dev/null 2>&1; echo "c3 rc=$?"
timeout -s KILL 900 $P -k regex:mha64 -s 2 -c 1 -o gpurun_out/m64_c5 python scripts/profile_forward.py --config c5 --iters 1 > /dev/null 2>&1; echo "c5 rc=$?"
for r in m64_c3 m64_c5; do
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
