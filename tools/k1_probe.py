import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig
from paper_2105_05821_b200.synth import synthetic_trace, synthetic_model
t = synthetic_trace(2_000_000, 101); m = synthetic_model(synthetic_trace(200_000, 101), 1)
g = GpuSimulator(0, "tf32x3"); g.load_model(m)
pc = ParallelConfig(k=1024)
g.load_trace(t, pc, oracle=True)
for ti in (False, True):
    r = g.run(pc, oracle=True, truth_inputs=ti)
    print("gather" if ti else "apply-only", round(r.device_ms, 1), "ms us/round", round(1000 * r.device_ms / r.rounds, 2))
g.load_trace(t, pc)
r = g.run(pc)
print("cnn", round(r.device_ms, 1), "us/round", round(1000 * r.device_ms / r.rounds, 2))
