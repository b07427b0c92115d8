#!/bin/bash
cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:mha2_fwd -s 2 -c 1 -o gpurun_out/mha2_c3 python scripts/one_kernel.py mha2 c3 > gpurun_out/ncu_mha2.log 2>&1
BT_MHA_V2=0 ncu --set full --import-source on --clock-control none -k regex:mha_fwd -s 2 -c 1 -o gpurun_out/mha1_c3 python scripts/one_kernel.py mha2 c3 > gpurun_out/ncu_mha1.log 2>&1
ls -la gpurun_out/*.ncu-rep
