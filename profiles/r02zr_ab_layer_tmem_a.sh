# Generic tensor-core layers (RB7-like model, residual C3) with A in tensor memory (3xTF32), same build:
# default vs SIMNET_LAYER_SS=1 (A from shared memory); tests of those paths
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "rb7 or residual or generic or layer" 2>&1 | tail -2
for i in 1 2; do for v in SIMNET_LAYER_SS=1 X=0; do
  env $v timeout 300 python profiles/rb7_prof.py tf32x3 | sed "s|^|[$v] |"
done; done
