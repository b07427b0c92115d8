cd $GRAFT_REPO_ROOT
for m in 0 6 7 8 1 2; do echo "== mode $m"; python scripts/gemm_trace.py 2458 3072 768 0 -256 $m | grep -E "event|finish|mainloop|epilogue per"; done
for m in 0 6 8; do echo "== bias PAIR1 256 mode $m"; python scripts/gemm_trace.py 2458 2304 768 1 256 $m | grep -E "finish|mainloop|epilogue per"; done
