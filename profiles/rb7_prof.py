import sys; sys.path.insert(0, ".")
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig
from paper_2105_05821_b200.formats import CnnConfig
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
cfg = CnnConfig.preset_rb7()
m = synthetic_model(synthetic_trace(200_000, 101), 1, config=cfg)
t = synthetic_trace(20_000, 101)
g = GpuSimulator(0, sys.argv[1]); g.load_model(m)
pc = ParallelConfig(k=1024, sim=SimConfig(max_context=cfg.max_context)); g.load_trace(t, pc)
r = g.run(pc)
print(f"rb7 {sys.argv[1]}: {r.rounds} rounds, {1e3 * r.device_ms / r.rounds:.1f} us/round, launches {r.launches}")
