# A/B: rounds per CUDA graph (SIMNET_GRAPH_ROUNDS); the remainder runs as one tail graph
for i in 1 2; do for G in 16 64 256; do
  echo "G=$G $(SIMNET_GRAPH_ROUNDS=$G timeout 120 python profiles/prof_run.py --runs 3)"
  echo "G=$G $(SIMNET_GRAPH_ROUNDS=$G timeout 120 python profiles/prof_run.py --runs 3 --precision bf16)"
  echo "G=$G $(SIMNET_GRAPH_ROUNDS=$G timeout 200 python profiles/prof_run.py --runs 2 --n 3000000 --k 1024)"
done; done
echo "base $(cd .ab/base && timeout 120 python profiles/prof_run.py --runs 3)"
echo "base $(cd .ab/base && timeout 200 python profiles/prof_run.py --runs 2 --n 3000000 --k 1024)"
