# Evidence for the round-2 kernels: the persistent FC kernel as ONE launch (ncu launch list + a full
# capture on a short c1 trace), and compute-sanitizer on the new paths.
mkdir -p gpurun_out
cat > /tmp/c1_short.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig
from paper_2105_05821_b200.formats import CnnConfig
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
cfg = CnnConfig.preset_fc2()
m = synthetic_model(synthetic_trace(200_000, 101), 1, config=cfg)
t = synthetic_trace(int(sys.argv[1]), 101)
g = GpuSimulator(0, "fp32"); g.load_model(m)
pc = ParallelConfig(k=1, sim=SimConfig(max_context=cfg.max_context)); g.load_trace(t, pc)
r = g.run(pc)
print(f"c1 short: {t.n} instructions, {r.launches} launch(es), {1e3 * r.device_ms / t.n:.2f} us per instruction")
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02p_c1_launches.csv \
   python /tmp/c1_short.py 20000 > gpurun_out/r02p_c1_short.txt 2>&1
python profiles/summarize_launches.py gpurun_out/r02p_c1_launches.csv > gpurun_out/r02p_c1_launches.txt 2>&1
cat gpurun_out/r02p_c1_short.txt gpurun_out/r02p_c1_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seq_fc -c 1 \
   -o gpurun_out/r02p_full_seq_fc python /tmp/c1_short.py 5000 > /dev/null 2>&1; echo "ncu full rc=$?"
python profiles/ncu_summary.py gpurun_out/r02p_full_seq_fc.ncu-rep > gpurun_out/r02p_seq_fc_ncu_summary.txt 2>&1
cat gpurun_out/r02p_seq_fc_ncu_summary.txt
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T python /tmp/c1_short.py 3000 2>&1 | tail -2 | sed "s/^/seq_fc $T: /"
done
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "multi_tile" 2>&1 | tail -2 | sed "s/^/fc1 multi-tile memcheck: /"
