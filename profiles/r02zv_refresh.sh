# r02zv final HEAD refresh on one B200 (FC1 A in TMEM for one-tile CTAs, generic layers A in TMEM, lazy sub_results)
# (tf32x3 / bf16 / fp8 / reference / trained weights / c3), launch lists, ncu --set full of the
# two round kernels, front phase trace, kernel spans, c1/c3/c4 configs, c2t parity per precision.
mkdir -p gpurun_out
T=r02zv
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
for P in tf32x3 bf16 fp8; do
  timeout 900 python bench.py --steps 3 --warmup 3 --precision $P $([ $P != tf32x3 ] && echo --no-cpu-baseline) \
     > gpurun_out/${T}_bench_$P.jsonl 2> gpurun_out/${T}_bench_$P.err; echo "bench $P rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.jsonl 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --weights trained --no-cpu-baseline > gpurun_out/${T}_bench_trained.jsonl 2> gpurun_out/${T}_bench_trained.err; echo "trained rc=$?"
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.jsonl 2> gpurun_out/${T}_bench_c3.err; echo "c3 rc=$?"
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
timeout 1800 python tools/configs.py --only c3,c4,rb7 > gpurun_out/${T}_configs.jsonl 2>&1; echo "configs rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_layer -s 20 -c 1 \
   -o gpurun_out/${T}_c3_full_tf32x3_tc_layer python profiles/prof_run.py --precision tf32x3 --k 8192 --n 300000 > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/${T}_c3_full_tf32x3_tc_layer.ncu-rep > gpurun_out/${T}_c3_ncu_fc1_summary.txt 2>&1
timeout 600 python tools/e2e_c3.py > gpurun_out/${T}_e2e_c3.txt 2>&1; timeout 300 python tools/e2e_breakdown.py > gpurun_out/${T}_e2e_c2.txt 2>&1
ls -la gpurun_out | tail -40
