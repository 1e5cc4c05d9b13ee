# diagnostics: fused round-front phase clocks in graph mode (SIMNET_CHAIN_TRACE=1)
import sys, ctypes as C, numpy as np, os
os.environ["SIMNET_CHAIN_TRACE"] = "1"
sys.path.insert(0, '/root/repo')
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, _lib
from paper_2105_05821_b200.synth import synthetic_trace, synthetic_model
N = int(os.environ.get("N", "300000")); t = synthetic_trace(N, 101)
K = int(os.environ.get("K", "1024")); NC = min(148, (K + 7) // 8)
m = synthetic_model(synthetic_trace(200_000, 101), 1)
for prec in os.environ.get("PRECS", "tf32x3,bf16").split(","):
    g = GpuSimulator(0, prec); g.load_model(m)
    pc = ParallelConfig(k=K); g.load_trace(t, pc); g.run(pc)
    W = 148 * 32 + 256 * 32 + 148 * 16
    full = np.zeros(W, np.int64)
    _lib.lib().simnet_debug_chain_trace_full(C.c_void_p(full.ctypes.data), C.c_int(W))
    buf = full[:148 * 32]
    tx = full[148 * 32 + 256 * 32:].reshape(148, 16)[:NC].astype(np.float64)
    tr = buf.reshape(148, 32)[:NC].astype(np.float64)
    T = tr[:, 20]
    base = tr[:, :1]
    names = {0: "start", 15: "dep wait done", 16: "apply done (warp0)", 1: "table done", 2: "tile0 gathered",
             3: "tile1 gathered", 6: "conv0 done", 7: "a1 tile0", 8: "a1 tile1", 9: "conv1 done", 10: "a2",
             11: "conv2 done", 12: "out done"}
    print(prec, "T histogram", np.bincount(T.astype(int)))
    ap = tr[:, 16:24] - base
    print(f"  apply per warp: median {np.median(ap):.0f}, max over warps median {np.median(ap.max(1)):.0f}")
    for i, n in ((24, "W2 landed w0"), (28, "h ready (synced)"), (25, "cta8 fc done w0"), (26, "decode done w0"), (27, "apply done w0")):
        col = (tr[:, i] - base[:, 0])[tr[:, i] > 0]
        if col.size: print(f"  {n:18s} median {np.median(col):8.0f} cyc   max {col.max():8.0f}")
    names.update({21: "fc1 barrier enter", 22: "fc1 barrier exit", 23: "fc1 MMAs done", 31: "fc1 partials written"})
    for i in (0, 15, 16, 1, 2, 3, 6, 7, 8, 9, 10, 11, 12, 21, 22, 23, 31):
        col = (tr[:, i] - base[:, 0])[tr[:, i] > 0]
        if col.size: print(f"  {names[i]:18s} median {np.median(col):8.0f} cyc   max {col.max():8.0f}")
    for i, n in ((5, "w0 table: before tg wait"), (6, "w0 table: tg ready"), (7, "w0 table: loop done"),
                 (10, "w0 gather start"), (8, "w0 tile0 loads first lane"), (11, "w0 tile0 loads lane 2"),
                 (9, "w0 tile0 loads last lane"), (0, "w0 tile0 loads done"), (1, "w0 tile0 stores done"), (2, "w0 tile1 loads done"),
                 (3, "w0 tile1 t0 wait done"), (4, "w0 tile1 stores done")):
        col = (tx[:, i] - base[:, 0])[tx[:, i] > 0]
        if col.size: print(f"  {n:24s} median {np.median(col):8.0f} cyc   max {col.max():8.0f}")
