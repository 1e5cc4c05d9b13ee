# Final HEAD check of round 2: GPU tests, smoke, default bench line, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02zz_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02zz_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02zz_bench.jsonl 2> gpurun_out/r02zz_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02zz_bench_reference.jsonl 2>&1; echo "ref rc=$?"
python -c "
import json
d = json.loads(open('gpurun_out/r02zz_bench.jsonl').read().strip().splitlines()[-1])
r = json.loads(open('gpurun_out/r02zz_bench_reference.jsonl').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'parity', d['parity']['cpi_error_percent'], 'frac', d['roofline']['frac'], 'hbm', d['roofline_hbm']['frac'], 'clocks', d['clocks'], 'launches', d['gpu_launches'])
print('reference', r['value'], r['cpu_baseline'].get('cores'), r.get('product_library_loaded'), 'e2e ratio', d['e2e']['value'] / r['value'])
"
