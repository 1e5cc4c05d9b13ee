# A/B: L2 persistence window over the flat conv output (default) vs none (SIMNET_L2_PERSIST=0)
for i in 1 2; do
  for P in tf32x3 bf16; do
    timeout 120 python profiles/prof_run.py --precision $P --runs 3
    SIMNET_L2_PERSIST=0 timeout 120 python profiles/prof_run.py --precision $P --runs 3 | sed 's/^/nopersist: /'
    timeout 200 python profiles/prof_run.py --precision $P --k 8192 --n 1000000 --runs 2
    SIMNET_L2_PERSIST=0 timeout 200 python profiles/prof_run.py --precision $P --k 8192 --n 1000000 --runs 2 | sed 's/^/nopersist: /'
  done
done
