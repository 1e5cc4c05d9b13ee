# c5 points on the c3 trace (100M instructions, one B200) after the lazy result objects: 65,536 / 262,144 / 1,048,576 sub-traces
for K in 65536 262144 1048576; do
  timeout 1500 python bench.py --config c3 --k $K --steps 2 --warmup 1 --no-cpu-baseline 2> gpurun_out/r02zw_c5_$K.err | tail -1 > gpurun_out/r02zw_c5_$K.jsonl
  python -c "import json; d=json.loads(open('gpurun_out/r02zw_c5_$K.jsonl').read()); print($K, round(d['value'],2), round(d['e2e']['value'],2), d['ms_per_step'], d.get('cpi'), d['config']['rounds'])"
done
