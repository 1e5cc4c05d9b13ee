# A/B: FC1 CTAs per (N tile, K split) group along M (SIMNET_FC1_GX; default = one M tile each at K=1024)
for i in 1 2; do
for G in 0 4 2; do
  echo "gx=$G"; SIMNET_FC1_GX=$G python profiles/prof_run.py --precision tf32x3 --n 1000000 --runs 2
  SIMNET_FC1_GX=$G SIMNET_FC1_SS=1 python profiles/prof_run.py --precision tf32x3 --n 1000000 --runs 2 | sed 's/^/SS /'
done; done
