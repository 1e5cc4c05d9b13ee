# diagnostics: the c3 workload end to end (100M instructions, 65,536 sub-traces, one GPU):
# load_trace (H2D + pack, not overlapped) vs run (device) vs simulate_parallel (overlapped upload)
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, SimConfig
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace
import bench

n = int(os.environ.get("N", "100000000"))
k = int(os.environ.get("K", "65536"))
t = synthetic_trace(n, 101)
m = synthetic_model(synthetic_trace(200_000, 101), 1)
g = GpuSimulator(0, "tf32x3")
g.load_model(m)
pc = ParallelConfig(k=k, sim=SimConfig(max_context=m.config.max_context))
pt = bench.pinned_trace(t)
fetch = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.load_trace(pt, pc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = g.run(pc, fetch_out=fetch)
    t2 = time.perf_counter()
    print(f"load_trace {1e3 * (t1 - t0):7.1f} ms | run {1e3 * (t2 - t1):7.1f} ms (device {r.device_ms:7.1f} ms)", flush=True)
for win in os.environ.get("WINS", "0").split(","):
    if win != "0":
        os.environ["SIMNET_WIN_ROUNDS"] = win
    else:
        os.environ.pop("SIMNET_WIN_ROUNDS", None)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = g.simulate_parallel(pt, pc, fetch_out=fetch)
        t1 = time.perf_counter()
        print(f"simulate_parallel (overlapped upload, win {win}) {1e3 * (t1 - t0):7.1f} ms -> "
              f"{n / (t1 - t0) / 1e6:.2f} MIPS, cycles {r.total_cycles}", flush=True)
