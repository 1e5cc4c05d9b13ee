# A/B on one box, same build: FC1's resident 3xTF32 weight slice loaded raw (64 KB) and split on chip
# (default) vs the host-split hi + lo planes (128 KB, SIMNET_FC1_HOST_SPLIT=1); then the GPU tests
for i in 1 2; do
  for v in "SIMNET_FC1_HOST_SPLIT=1" "X=0"; do
    env $v timeout 120 python profiles/prof_run.py --precision tf32x3 --runs 3 2>&1 | sed "s|^|[$v] |"
    env $v timeout 200 python profiles/prof_run.py --precision tf32x3 --k 8192 --n 1000000 --runs 2 2>&1 | sed "s|^|[$v] |"
  done
done
PRECS=tf32x3 timeout 300 python tools/fc1_trace.py 2>&1 | head -14
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02zg_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02zg_pytest.log
