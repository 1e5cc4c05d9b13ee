# diagnostics: FC1 (tc_layer_kernel) per-CTA event clocks in graph mode (SIMNET_CHAIN_TRACE=1)
import ctypes as C
import os
import sys

import numpy as np

os.environ["SIMNET_CHAIN_TRACE"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, _lib  # noqa: E402
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace  # noqa: E402

K = int(os.environ.get("K", "1024"))
t = synthetic_trace(max(300_000, 300 * K), 101)
m = synthetic_model(synthetic_trace(200_000, 101), 1)
for prec in os.environ.get("PRECS", "tf32x3,bf16").split(","):
    g = GpuSimulator(0, prec)
    g.load_model(m)
    pc = ParallelConfig(k=K)
    g.load_trace(t, pc)
    g.run(pc)
    buf = np.zeros(148 * 32 + 256 * 32, np.int64)
    _lib.lib().simnet_debug_chain_trace_full(C.c_void_p(buf.ctypes.data), C.c_int(buf.size))
    tr = buf[148 * 32:].reshape(256, 32)[:128].astype(np.float64)
    rel = tr - tr[:, :1]
    names = {0: "start", 1: "W landed", 11: "split: chunk0 landed", 29: "split: chunk0 in TMEM", 30: "split: chunk1 landed",
             31: "split: chunk1 in TMEM", 2: "A chunk0 ready", 5: "A chunk1 ready", 6: "A chunk2 ready",
             7: "A chunk3 ready", 3: "tile0 MMAs issued", 14: "accumulator done", 16: "epi: tmem ld", 17: "epi: staged",
             18: "epi: fenced", 19: "epi: TMA issued", 20: "epi: staging read", 4: "tile0 epilogue done"}
    print(prec)
    dw = (tr[:, 12] - tr[:, 8]) * 1.87
    print(f"  MMA issue total      median {np.median(tr[:, 15]):8.0f} cyc")
    print(f"  dependency wait exit median {np.median(dw):8.0f} cyc (globaltimer x 1.87)")
    per = rel[:, 21:29]
    ok = per[:, 1:] > 0
    if ok.any():
        d = np.diff(per, axis=1)[ok]
        print(f"  tile MMA-issue period (tiles 1..7) median {np.median(d):8.0f} cyc")
        print("  tile issue times (median over CTAs):", " ".join(f"{np.median(per[:, i][per[:, i] > 0]):.0f}"
                                                          for i in range(8) if (per[:, i] > 0).any()))
    for i, n in names.items():
        col = rel[:, i][tr[:, i] > 0]
        if col.size:
            print(f"  {n:20s} median {np.median(col):8.0f} cyc   max {col.max():8.0f}")
