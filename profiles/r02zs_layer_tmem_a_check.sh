# generic layers with A in tensor memory: full GPU suite, RB7 at-scale parity (tf32x3), RB7 timing both precisions
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02zs_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02zs_pytest.log
timeout 1200 python tools/scale_parity.py gpu --only rb7 --precisions tf32x3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['workload'], d['precision'], '%.4f%%' % d['cpi_error_percent'], d.get('subtrace_identical_frac'), round(d.get('fetch_block_identical_frac', 0), 4), '%.3f MIPS' % d['gpu_mips'])
"
for P in tf32x3 bf16; do timeout 300 python profiles/rb7_prof.py $P; done
