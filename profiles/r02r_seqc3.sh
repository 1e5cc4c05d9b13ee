# Persistent C3 at one sub-trace (seq_c3_kernel): GPU tests, timing vs the launch-per-layer rounds and tf32x3 K=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fc2.py -m gpu -q -p no:cacheprovider -k "persistent" 2>&1 | tail -4
timeout 300 python profiles/prof_run.py --precision fp32 --k 1 --n 20000
SIMNET_NO_SEQ_FC=1 timeout 300 python profiles/prof_run.py --precision fp32 --k 1 --n 20000 | sed 's/^/launch-per-layer: /'
timeout 300 python profiles/prof_run.py --precision tf32x3 --k 1 --n 20000 | sed 's/^/tf32x3 fused: /'
timeout 300 python profiles/prof_run.py --precision fp32 --k 1 --n 20000 --model tests/golden/c3_trained.model | sed 's/^/trained: /'
