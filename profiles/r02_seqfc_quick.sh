timeout 600 python -m pytest tests/test_fc2.py -m gpu -x -q -p no:cacheprovider -k persistent 2>&1 | tail -2
SIMNET_SEQ_TRACE=1 timeout 900 python tools/configs.py --only c1 --c1-n 200000 2>&1 | tail -2
