# racecheck details on the persistent FC kernel (short trace)
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
print(f"c1 short: {t.n} instructions, {r.launches} launch(es)")
PY
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python /tmp/c1_short.py 300 > gpurun_out/r02q_racecheck.txt 2>&1
grep -E "Warning|Error|hazard|at 0x|in .*cu:|RACECHECK" gpurun_out/r02q_racecheck.txt | sort | uniq -c | sort -rn | head -40
