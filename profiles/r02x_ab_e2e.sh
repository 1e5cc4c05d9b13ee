# A/B: e2e (simulate_parallel, pinned host buffers) with the geometric first upload windows
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "overlapped or chunked or write_ring" 2>&1 | tail -2
for i in 1 2; do
  for d in .ab/base .; do
    (cd $d && timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$d', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))")
  done
done
