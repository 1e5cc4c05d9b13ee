# diagnostics: where the e2e time goes (load_trace = H2D + pack; run = capture + rounds + D2H)
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
import bench

n = 10_000_000
t = synthetic_trace(n, 101)
m = synthetic_model(synthetic_trace(200_000, 101), 1)
g = GpuSimulator(0, "tf32x3")
g.load_model(m)
pc = ParallelConfig(k=1024, sim=SimConfig(max_context=m.config.max_context))
pt = bench.pinned_trace(t)
import numpy as np
fetch = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
for rep in range(6):
    out = fetch if rep >= 3 else None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.load_trace(pt, pc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = g.run(pc, fetch_out=out)
    t2 = time.perf_counter()
    print(f"load_trace {1e3 * (t1 - t0):7.1f} ms | run {1e3 * (t2 - t1):7.1f} ms (device {r.device_ms:7.1f} ms) | "
          f"total {1e3 * (t2 - t0):7.1f} ms -> {n / (t2 - t0) / 1e6:.2f} MIPS {'(pinned fetch_out)' if out is not None else ''}")

for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = g.simulate_parallel(pt, pc, fetch_out=fetch)
    t1 = time.perf_counter()
    print(f"simulate_parallel (overlapped upload) {1e3 * (t1 - t0):7.1f} ms -> {n / (t1 - t0) / 1e6:.2f} MIPS, "
          f"cycles {r.total_cycles}")
