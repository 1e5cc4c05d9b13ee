# A/B: FC1 A-ring depth for CTAs looping over M tiles (c3 shard, K = 8192): 4 (default) / 5 / 6 stages
for i in 1 2; do
  for P in tf32x3 bf16; do
    for N in 4 5 6; do
      SIMNET_FC1_STAGES=$N timeout 200 python profiles/prof_run.py --precision $P --k 8192 --n 1000000 --runs 2 | sed "s/^/stages $N: /"
    done
  done
done
SIMNET_FC1_STAGES=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "multi_tile" 2>&1 | tail -2
