# A/B: FC1 CTAs looping over M tiles, TMA-stored partial tiles (default) vs per-thread row stores
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "multi_tile or tma_store" 2>&1 | tail -3
for P in tf32x3 bf16; do
  for rep in 1 2; do
    timeout 300 python profiles/prof_run.py --precision $P --n 1000000 --k 8192 --runs 2
    SIMNET_FC1_MULTI_DIRECT=1 timeout 300 python profiles/prof_run.py --precision $P --n 1000000 --k 8192 --runs 2 | sed 's/^/direct: /'
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv \
   --log-file gpurun_out/r02j_c3_launches_tf32x3.csv python profiles/prof_run.py --precision tf32x3 --n 1000000 --k 8192 > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/r02j_c3_launches_tf32x3.csv
