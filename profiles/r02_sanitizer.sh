# compute-sanitizer memcheck / synccheck on smoke() and the round-2 GPU tests (one B200)
CS=/usr/local/cuda/bin/compute-sanitizer
K="rb7 or device_group or write_ring_grows or decode_goldens_on_device or fused_front"
timeout 900 $CS --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_memcheck_smoke.txt 2>&1; echo "memcheck smoke rc=$?"
timeout 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py -k "$K" > gpurun_out/r02h_memcheck_tests.txt 2>&1; echo "memcheck tests rc=$?"
timeout 900 $CS --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_synccheck_smoke.txt 2>&1; echo "synccheck smoke rc=$?"
for f in gpurun_out/r02h_*.txt; do echo "== $f"; tail -n 3 $f; done
