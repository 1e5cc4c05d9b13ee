for i in 1 2; do
python profiles/prof_run.py --precision tf32x3 --n 1000000 --runs 2
SIMNET_DIAG_FC1_SKIP_W=1 python profiles/prof_run.py --precision tf32x3 --n 1000000 --runs 2
done
