# Streamed weights for large-M conv layers (RB7): tests, timing A/B vs split-K, scale parity
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "rb7 or residual" 2>&1 | tail -3
for P in tf32x3 bf16; do
  timeout 300 python profiles/rb7_prof.py $P
  SIMNET_NO_STREAM_W=1 timeout 300 python profiles/rb7_prof.py $P | sed 's/^/split-K: /'
done
timeout 1200 python tools/scale_parity.py gpu --only rb7 --precisions tf32x3,bf16 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['workload'], d['precision'], '%.4f%%' % d['cpi_error_percent'], d.get('subtrace_identical_frac'), round(d.get('fetch_block_identical_frac', 0), 4), '%.3f MIPS' % d['gpu_mips'])
"
