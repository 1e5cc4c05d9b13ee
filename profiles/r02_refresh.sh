# r02 HEAD refresh on one B200: bench lines (tf32x3 / bf16 / fp8), launch lists,
# ncu --set full captures of the two round kernels, the front phase trace and
# the c3 / c4 configs.  Run under gpurun; outputs in gpurun_out/, summaries
# copied to profiles/r02*.
mkdir -p gpurun_out
T=${TAG:-r02d}
for P in tf32x3 bf16 fp8; do
  timeout 900 python bench.py --steps 3 --warmup 3 --precision $P $([ $P != tf32x3 ] && echo --no-cpu-baseline) \
     > gpurun_out/${T}_bench_$P.jsonl 2> gpurun_out/${T}_bench_$P.err; echo "bench $P rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.jsonl 2>&1; echo "ref rc=$?"
for P in tf32x3 bf16; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 200 --csv \
     --log-file gpurun_out/${T}_launches_$P.csv python profiles/prof_run.py --precision $P > /dev/null 2>&1
  python profiles/summarize_launches.py gpurun_out/${T}_launches_$P.csv > gpurun_out/${T}_launches_$P.txt 2>&1
done
for K in round_front tc_layer; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 40 -c 1 \
     -o gpurun_out/${T}_full_tf32x3_$K python profiles/prof_run.py --precision tf32x3 --n 100000 > /dev/null 2>&1
  echo "ncu $K rc=$?"
done
python profiles/ncu_summary.py gpurun_out/${T}_full_tf32x3_*.ncu-rep > gpurun_out/${T}_ncu_full_summary.txt 2>&1
PRECS=tf32x3,bf16 timeout 600 python tools/front_trace.py > gpurun_out/${T}_front_trace.txt 2>&1
PRECS=tf32x3 timeout 600 python tools/kernel_spans.py > gpurun_out/${T}_kernel_spans.txt 2>&1
timeout 1200 python tools/configs.py --only c3,c4 > gpurun_out/${T}_configs.jsonl 2>&1; echo "configs rc=$?"
ls -la gpurun_out | tail -30
