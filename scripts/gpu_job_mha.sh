# MHA A/B: GPU suite on the working tree, then MHA launch timing per library variant.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for r in 1 2; do
for v in base=scripts/ab/base.so new=default ${EXTRA_VARIANTS}; do
  name=${v%%=*}; lib=${v#*=}; [ "$lib" = "default" ] && lib=""
  BT_LIB_PATH=$lib timeout -s KILL 300 python scripts/mha_time.py c2 c3 c5 2>&1 | sed "s/^/$name /"
done; done
