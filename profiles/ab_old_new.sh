# A/B of older commits (git worktrees under .ab/, built locally) against HEAD on the same box
for i in 1 2; do
  for d in .ab/*; do (cd $d && timeout 60 python profiles/prof_run.py --precision tf32x3 --runs 3 | sed "s|^|$d |"); done
  timeout 60 python profiles/prof_run.py --precision tf32x3 --runs 3 | sed 's/^/HEAD /'
done
