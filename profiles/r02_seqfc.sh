# Persistent FC kernel (seq_fc.cu): GPU tests, c1 at 1M instructions, A/B vs the launch-per-layer rounds
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fc2.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 900 python tools/configs.py --only c1 2>&1 | tail -3
SIMNET_NO_SEQ_FC=1 timeout 900 python tools/configs.py --only c1 --c1-n 100000 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_fc2.py -m gpu -x -q -p no:cacheprovider -k "persistent and 1" 2>&1 | tail -6
