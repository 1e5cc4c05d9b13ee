# same-box A/B of .ab/base vs HEAD for tf32x3, bf16, fp8 (K=1024) and tf32x3 c3
for i in 1 2; do
  for d in .ab/base .; do
    for P in tf32x3 bf16 fp8; do echo "$d $(cd $d && timeout 120 python profiles/prof_run.py --precision $P --runs 3)"; done
    echo "$d $(cd $d && timeout 200 python profiles/prof_run.py --runs 3 --n 2000000 --k 8192)"
  done
done
