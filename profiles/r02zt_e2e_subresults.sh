# lazy ParallelResult.sub_results (numpy-backed): GPU suite, the c3 end-to-end breakdown, bench c3 line
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02zt_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02zt_pytest.log
timeout 900 python tools/e2e_c3.py 2>&1 | tail -4
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02zt_bench_c3.jsonl 2> gpurun_out/r02zt_bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02zt_bench.jsonl 2> gpurun_out/r02zt_bench.err; echo "bench rc=$?"
python -c "
import json
for f in ('gpurun_out/r02zt_bench_c3.jsonl', 'gpurun_out/r02zt_bench.jsonl'):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d['value'], d['e2e']['value'], d['parity'].get('cpi_error_percent'), d['clocks'])
"
