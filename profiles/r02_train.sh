# Train the C3 on the GPU (tests/golden/train_c3.py: reference DES traces + truth-latency requests,
# reference loss, Adam, DAgger-style closed-loop aggregation, closed-loop validation selects the
# epoch), then the round cost with the trained model
mkdir -p gpurun_out
timeout 3000 python tests/golden/train_c3.py --n-per-trace 60000 --seeds 4 --epochs 20 --dagger 4000 --out gpurun_out/c3_trained.model 2>&1 | tail -35
for P in tf32x3 bf16; do
  timeout 300 python profiles/prof_run.py --precision $P --runs 2 --model gpurun_out/c3_trained.model
  timeout 300 python profiles/prof_run.py --precision $P --runs 2 --k 8192 --n 1000000 --model gpurun_out/c3_trained.model
done
