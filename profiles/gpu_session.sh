set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_tf32x3.log 2>&1
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1
tail -3 gpurun_out/*.log
