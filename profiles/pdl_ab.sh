# PDL per launch tag (same binary): none / layer (FC1) / front / both
for i in 1 2; do for P in tf32x3 bf16; do for V in 0 layer front layer,front; do
  SIMNET_PDL=$V timeout 60 python profiles/prof_run.py --precision $P --runs 3 | sed "s/^/PDL=$V /"
done; done; done
