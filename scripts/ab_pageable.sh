# A/B of the pageable-input host paths (BT_PAGEABLE_STAGE) at C2 + their parity tests
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_encoder.py tests/test_service.py -x -q > gpurun_out/pageable_tests.txt 2>&1
echo TEST_RC=$? >> gpurun_out/pageable_tests.txt
for i in 1 2 3; do
 for v in 0 1; do
  BT_PAGEABLE_STAGE=$v timeout 300 python scripts/e2e_numpy_profile.py 2>/dev/null | head -1 | sed "s/^/STAGE=$v /"
  BT_PAGEABLE_STAGE=$v timeout 300 python scripts/stream_numpy_probe.py 2>/dev/null | sed "s/^/STAGE=$v /"
 done
done
