# A/B on one box: .ab/base (previous commit, built locally) vs the working tree
# (FC1 one-tile CTAs: partials by coalesced generic stores from the staging);
# c2 shape (K = 1024) and the c3 shard shape (K = 8192), tf32x3 and bf16; then GPU tests
for i in 1 2; do
  for d in .ab/base .; do
    (cd $d && for p in tf32x3 bf16; do
       timeout 120 python profiles/prof_run.py --precision $p --runs 3
       timeout 200 python profiles/prof_run.py --precision $p --k 8192 --n 1000000 --runs 2
     done) 2>&1 | sed "s|^|$d |"
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02zq_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02zq_pytest.log
