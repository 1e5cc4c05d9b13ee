import sys, ctypes as C, numpy as np, os
os.environ["SIMNET_CHAIN_TRACE"] = "1"
sys.path.insert(0, '/root/repo')
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, _lib
from paper_2105_05821_b200.synth import synthetic_trace, synthetic_model
t = synthetic_trace(300_000, 101); m = synthetic_model(synthetic_trace(200_000, 101), 1)
for prec in ("tf32x3", "bf16"):
    g = GpuSimulator(0, prec); g.load_model(m)
    pc = ParallelConfig(k=1024); g.load_trace(t, pc); g.run(pc, profile=True)
    buf = np.zeros(148 * 32, np.int64)
    _lib.lib().simnet_debug_chain_trace(C.c_void_p(buf.ctypes.data))
    tr = buf.reshape(148, 32)[:128, :14].astype(np.float64)
    rel = tr - tr[:, :1]
    names = ["start","W0 issued","c0 seen(prod)","m1b seen(prod)","W0 ready(mma)","conv0 issued","a0 ready","W1 ready","a1 ready","a2 ready","W2 ready","conv2 issued","m2 seen(epi)","out done"]
    print(prec)
    for i, n in enumerate(names):
        print(f"  {n:16s} median {np.median(rel[:, i]):8.0f} cyc   max {rel[:, i].max():8.0f}")
