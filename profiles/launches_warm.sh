# per-kernel device time, warm caches (ncu --cache-control none), serialized launches
mkdir -p gpurun_out
for P in tf32x3 bf16; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 400 -c 200 --csv \
     --log-file gpurun_out/lw_$P.csv python profiles/prof_run.py --precision $P > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 400 -c 200 --csv \
     --log-file gpurun_out/lw_${P}_unfused.csv python profiles/prof_run.py --precision $P --unfused > /dev/null 2>&1
done
for f in gpurun_out/lw_*.csv; do echo "== $f"; python profiles/summarize_launches.py $f; done
