# A/B: FC1 weight-slice multicast cluster size (SIMNET_FC1_MCAST), same box
for i in 1 2; do
for M in 1 2 4 8; do
  echo "mcast=$M"; SIMNET_FC1_MCAST=$M python profiles/prof_run.py --precision tf32x3 --n 1000000 --runs 2
done
done
for M in 1 2 4; do
  echo "mcast=$M K=8192"; SIMNET_FC1_MCAST=$M python profiles/prof_run.py --precision tf32x3 --n 1000000 --k 8192 --runs 2
  echo "mcast=$M bf16"; SIMNET_FC1_MCAST=$M python profiles/prof_run.py --precision bf16 --n 1000000 --runs 2
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
