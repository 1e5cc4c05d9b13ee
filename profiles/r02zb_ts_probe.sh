# tcgen05.mma issue cost with A from tensor memory (FC1's form at c3) next to the SMEM form
mkdir -p gpurun_out
timeout 300 python tools/probes/tc_peak.py --no-dense > gpurun_out/r02zb_ts_probe.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r02zb_ts_probe.txt
