cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
 for m in padded staged; do
  BT_STREAM_PAGEABLE=$m timeout 300 python scripts/stream_numpy_probe.py 2>/dev/null | sed "s/^/MODE=$m /"
 done
done
BT_STREAM_PAGEABLE=padded timeout 300 python scripts/stream_numpy_probe.py --trace 2>&1 | tail -3
