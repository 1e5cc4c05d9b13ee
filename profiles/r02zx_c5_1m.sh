# c5 at 1,048,576 sub-traces after the partition starts stay a numpy array on the hot path; GPU tests
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02zx_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02zx_pytest.log
for K in 1048576 65536; do
  timeout 1500 python bench.py --config c3 --k $K --steps 2 --warmup 1 --no-cpu-baseline 2> gpurun_out/r02zx_c5_$K.err | tail -1 > gpurun_out/r02zx_c5_$K.jsonl
  python -c "import json; d=json.loads(open('gpurun_out/r02zx_c5_$K.jsonl').read()); print($K, round(d['value'],2), round(d['e2e']['value'],2), d['ms_per_step'], d.get('cpi'), d['config']['rounds'])"
done
