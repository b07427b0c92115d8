#!/bin/bash
# L2 traffic of the C2 GEMMs per tile shape (ncu, cold single launches after warm-up)
cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum"
for cfg in "2458 2304 768 1 192" "2458 2304 768 1 -256" "2458 3072 768 2 -256" "2458 3072 768 2 256" "2458 768 3072 0 -128" "2458 768 768 0 128" "4917 3072 1024 1 -256"; do
  ncu --metrics $M --clock-control none -k regex:gemm_bf16 -s 2 -c 1 --csv python scripts/one_kernel.py gemm $cfg > gpurun_out/ncu_l2_$(echo $cfg | tr ' ' '_').csv 2>&1
done
