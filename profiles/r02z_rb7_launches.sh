# RB7-like model: launch list of one run (20k instructions, K = 1024), tf32x3 and bf16
for P in tf32x3 bf16; do
  timeout 300 python profiles/rb7_prof.py $P
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv \
     --log-file gpurun_out/r02z_rb7_launches_$P.csv python profiles/rb7_prof.py $P > /dev/null 2>&1
  python profiles/summarize_launches.py gpurun_out/r02z_rb7_launches_$P.csv
done
