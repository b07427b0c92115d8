# mha64 persistent item mapping: sibling tiles on one CTA (default) vs unit stride (abvar/sib0)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_configs.py tests/test_gpu_determinism.py tests/test_gpu_encoder.py -q -x > gpurun_out/sib_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/sib_tests.txt
for r in 1 2; do
 for v in sib1 sib0; do
  [ $v = sib0 ] && lib=abvar/sib0/libbt200.so || lib=""
  BT_LIB_PATH=$lib timeout -s KILL 500 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'], {k: round(v['us'],1) for k, v in d['kernels'].items() if k in ('mha',)})"
 done
done
timeout 600 ncu --profile-from-start off --clock-control none -k regex:mha64 -c 1 --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --csv python scripts/profile_forward.py --config c5 --iters 1 > gpurun_out/mha_l2_sib.csv 2>/dev/null; grep -v "^==" gpurun_out/mha_l2_sib.csv | cut -d, -f13- | tail -3
