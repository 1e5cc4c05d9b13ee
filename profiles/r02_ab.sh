# A/B of .ab/* worktrees (older commits, built locally) against the working tree, same box
for i in 1 2; do
  for d in .ab/*; do (cd $d && for p in tf32x3 bf16; do timeout 60 python profiles/prof_run.py --precision $p --n 1000000 --runs 2 | sed "s|^|$d |"; done; timeout 100 python profiles/prof_run.py --precision tf32x3 --k 8192 --n 2000000 --runs 2 | sed "s|^|$d |"); done
  for p in tf32x3 bf16; do timeout 60 python profiles/prof_run.py --precision $p --n 1000000 --runs 2 | sed 's/^/HEAD /'; done
  timeout 100 python profiles/prof_run.py --precision tf32x3 --k 8192 --n 2000000 --runs 2 | sed 's/^/HEAD /'
done
