# One GPU session: tests, bench lines (ours tf32x3 / bf16, reference arm), launch lists and ncu captures.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_tf32x3.log 2>&1; tail -1 gpurun_out/bench_tf32x3.log
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1; tail -1 gpurun_out/bench_bf16.log
timeout 600 python bench.py --precision fp8 --no-cpu-baseline > gpurun_out/bench_fp8.log 2>&1; tail -1 gpurun_out/bench_fp8.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; tail -1 gpurun_out/bench_reference.log
for P in tf32x3 bf16; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 200 --csv \
     --log-file gpurun_out/launches_$P.csv python profiles/prof_run.py --precision $P > /dev/null 2>&1
  for K in round_front tc_layer; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
       -o gpurun_out/full_${P}_$K python profiles/prof_run.py --precision $P --n 100000 > /dev/null 2>&1
  done
done
ls gpurun_out
