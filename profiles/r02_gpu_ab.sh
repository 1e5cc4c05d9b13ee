# r02: GPU tests, then the c2 bench and the tf32x3 scale parity (A/B vs the previous commit's numbers)
set -o pipefail
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02c_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02c_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench.json 2>gpurun_out/r02c_bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02c_bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'front_us', d['roofline']['launch_us'], 'kern', d['kernels_ms_per_step'], 'parity', d['parity']['rel_err'], d['parity']['fetch_block_identical_frac'])"
timeout 900 python tools/scale_parity.py gpu --only c2,c4,c3s --precisions tf32x3 > gpurun_out/r02c_parity.jsonl 2>&1; echo "parity rc=$?"
python -c "
import json
for l in open('gpurun_out/r02c_parity.jsonl'):
    d=json.loads(l); print(d['workload'],d['precision'],'%.4f%%'%d['cpi_error_percent'],d.get('subtrace_identical_frac'),round(d.get('fetch_block_identical_frac',0),4),'%.2f MIPS'%d['gpu_mips'],'%.1f us/round'%d['us_per_round'])
"
