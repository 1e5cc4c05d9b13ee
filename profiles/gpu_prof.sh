# launch list + ncu --set full captures of the round kernels (run under gpurun)
set -x
mkdir -p gpurun_out
P=${P:-tf32x3}
python profiles/prof_run.py --precision $P > gpurun_out/prof_plain_$P.log 2>&1
# rounds are graphs of 16; skip the first 400 launches (load, warm-up)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 200 --csv \
   --log-file gpurun_out/launches_$P.csv python profiles/prof_run.py --precision $P > /dev/null 2>&1
for K in conv_chain fc_tail ctx_kernel tc_layer; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 2 \
     -o gpurun_out/full_${P}_$K python profiles/prof_run.py --precision $P --n 100000 > /dev/null 2>&1
done
ls -la gpurun_out
