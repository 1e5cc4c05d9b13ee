# FC1 at the c3 shard shape after the warp-issued MMAs: per-tile clocks, and the A-in-SMEM / ring-depth knobs again
K=8192 PRECS=tf32x3,bf16 timeout 300 python tools/fc1_trace.py 2>&1 | tail -40
for v in "" "SIMNET_FC1_SS=1" "SIMNET_FC1_STAGES=5" "SIMNET_FC1_GX=12" "SIMNET_FC1_GX=6"; do
  env $v timeout 200 python profiles/prof_run.py --precision tf32x3 --k 8192 --n 1000000 --runs 2 2>&1 | sed "s|^|[$v] |"
done
