# c3 shard (K=8192) launch list: front vs FC1 per round, tf32x3 and bf16; plain timing too
mkdir -p gpurun_out
T=${TAG:-r02i}
for P in tf32x3 bf16; do
  timeout 300 python profiles/prof_run.py --precision $P --n 1000000 --k 8192 > gpurun_out/${T}_c3_time_$P.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv \
     --log-file gpurun_out/${T}_c3_launches_$P.csv python profiles/prof_run.py --precision $P --n 1000000 --k 8192 > /dev/null 2>&1
  python profiles/summarize_launches.py gpurun_out/${T}_c3_launches_$P.csv > gpurun_out/${T}_c3_launches_$P.txt 2>&1
  cat gpurun_out/${T}_c3_time_$P.txt gpurun_out/${T}_c3_launches_$P.txt
done
