for P in tf32x3 bf16; do for PDL in 0 1; do
  if [ $PDL = 1 ]; then export SIMNET_PDL=1; else unset SIMNET_PDL; fi
  timeout 120 python profiles/prof_run.py --precision $P --runs 2 | sed "s/^/PDL=$PDL /"
  timeout 120 python profiles/prof_run.py --precision $P --runs 2 --unfused | sed "s/^/PDL=$PDL /"
done; done
SIMNET_PDL=1 timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
