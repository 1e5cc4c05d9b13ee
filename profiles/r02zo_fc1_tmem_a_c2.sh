# c2 (one M tile per FC1 CTA): A from tensor memory (SIMNET_FC1_TMEM_A=1) vs A from shared memory, same build
for i in 1 2; do for v in X=0 SIMNET_FC1_TMEM_A=1; do
  env $v timeout 120 python profiles/prof_run.py --precision tf32x3 --runs 3 | sed "s|^|[$v] |"
done; done
SIMNET_FC1_TMEM_A=1 PRECS=tf32x3 timeout 300 python tools/fc1_trace.py 2>&1 | head -14
SIMNET_FC1_TMEM_A=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fused or fc1 or bench_workload" 2>&1 | tail -2
