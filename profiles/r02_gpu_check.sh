set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r02a_smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02a_bench_c2.json 2> gpurun_out/r02a_bench_c2.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02a_bench_c2.json
