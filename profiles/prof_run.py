"""Short, profiler-friendly run of the bench workload shape (C3, K sub-traces,
synthetic trace) for ncu launch lists and --set full captures.

  python profiles/prof_run.py [--precision tf32x3] [--n 300000] [--k 1024] [--regime default]

Numbers printed under a profiler are never bench values.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig  # noqa: E402
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--precision", default="tf32x3")
p.add_argument("--n", type=int, default=300_000)
p.add_argument("--k", type=int, default=1024)
p.add_argument("--regime", default="default")
p.add_argument("--runs", type=int, default=1)
p.add_argument("--unfused", action="store_true")
p.add_argument("--model", default=None, help="ILMD model file instead of the synthetic one")
a = p.parse_args()
kind = "memory" if a.regime == "memory" else "mix"
t = synthetic_trace(a.n, 101, kind=kind)
if a.model:
    from paper_2105_05821_b200 import read_model
    m = read_model(a.model)
else:
    m = synthetic_model(synthetic_trace(200_000, 101, kind=kind), 1, regime=a.regime)
g = GpuSimulator(0, a.precision)
g.load_model(m)
pc = ParallelConfig(k=a.k, sim=SimConfig(max_context=m.config.max_context))
g.load_trace(t, pc)
for _ in range(a.runs):
    r = g.run(pc, fused=not a.unfused)
import os
print(f"{a.precision}{' unfused' if a.unfused else ''}{' ' + a.model if a.model else ''} n={a.n} k={a.k}: "
      f"{r.rounds} rounds, {r.device_ms:.1f} ms, CPI {r.total_cycles / a.n:.4f}, "
      f"{1000 * r.device_ms / max(r.rounds, 1):.2f} us/round, launches {r.launches}")
