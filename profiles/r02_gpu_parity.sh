# r02: GPU tests + BASELINE-scale parity of every precision vs the reference fixtures
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
#timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?"
#tail -5 gpurun_out/r02b_pytest.log
timeout 1500 python tools/scale_parity.py gpu --only c2,c4,c3s > gpurun_out/r02b_parity.jsonl 2> gpurun_out/r02b_parity.err; echo "parity rc=$?"
cut -c1-400 gpurun_out/r02b_parity.jsonl
