# ncu --set full of the two round kernels at the c3 shard size (K = 8192), tf32x3
mkdir -p gpurun_out
T=${TAG:-r02k}
for K in round_front tc_layer; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
     -o gpurun_out/${T}_c3_full_tf32x3_$K python profiles/prof_run.py --precision tf32x3 --n 400000 --k 8192 > /dev/null 2>&1
  echo "ncu $K rc=$?"
done
python profiles/ncu_summary.py gpurun_out/${T}_c3_full_tf32x3_*.ncu-rep > gpurun_out/${T}_c3_ncu_full_summary.txt 2>&1
cat gpurun_out/${T}_c3_ncu_full_summary.txt
