# diagnostics: in-graph spans of the last round's two kernels from %globaltimer
# (SIMNET_CHAIN_TRACE=1): first CTA start .. last CTA end, and the gaps.
import ctypes as C
import os
import sys

import numpy as np

os.environ["SIMNET_CHAIN_TRACE"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2105_05821_b200 import GpuSimulator, ParallelConfig, _lib  # noqa: E402
from paper_2105_05821_b200.synth import synthetic_model, synthetic_trace  # noqa: E402

t = synthetic_trace(300_000, 101)
m = synthetic_model(synthetic_trace(200_000, 101), 1)
for prec in os.environ.get("PRECS", "tf32x3,bf16").split(","):
    g = GpuSimulator(0, prec)
    g.load_model(m)
    pc = ParallelConfig(k=1024)
    g.load_trace(t, pc)
    r = g.run(pc)
    W = 148 * 32 + 256 * 32
    buf2 = np.zeros(2 * W, np.int64)
    _lib.lib().simnet_debug_chain_trace_full(C.c_void_p(buf2.ctypes.data), C.c_int(buf2.size))
    buf = buf2[:W]
    nfr = buf2[W:W + 148 * 32].reshape(148, 32)[:128]  # the next round's front
    fr = buf[:148 * 32].reshape(148, 32)[:128]
    f1 = buf[148 * 32:].reshape(256, 32)[:128]
    fs, fe = fr[:, 13].min(), fr[:, 14].max()
    cs, ce = f1[:, 8].min(), f1[:, 9].max()
    per_round = 1000 * r.device_ms / r.rounds
    print(f"{prec}: round {per_round:.2f} us | front span {(fe - fs) / 1e3:.2f} us (CTA end spread "
          f"{(fr[:, 14].max() - np.median(fr[:, 14])) / 1e3:.2f}) | gap front->fc1 {(cs - fe) / 1e3:.2f} us | "
          f"fc1 span {(ce - cs) / 1e3:.2f} us | gap fc1->next front {per_round - (ce - fs) / 1e3:.2f} us (by subtraction)")
    # clock64 vs globaltimer on the same CTA span (sanity): front marks 0 (start) .. 12 (out done)
    cyc = (fr[:, 12] - fr[:, 0]).astype(np.float64)
    ns = (fr[:, 14] - fr[:, 13]).astype(np.float64)
    print(f"   front per-CTA: clock64 {np.median(cyc):.0f} cyc vs globaltimer {np.median(ns):.0f} ns -> "
          f"{np.median(cyc) / max(np.median(ns), 1):.3f} cyc/ns")
    cyc1 = (f1[:, 4] - f1[:, 0]).astype(np.float64)
    ns1 = (f1[:, 9] - f1[:, 8]).astype(np.float64)
    print(f"   fc1 per-CTA: clock64 {np.median(cyc1):.0f} cyc vs globaltimer {np.median(ns1):.0f} ns")
    dw = f1[:, 12]
    print(f"   timeline (ns from first front CTA start): front CTA ends median {np.median(fr[:, 14]) - fs:.0f} "
          f"max {fe - fs:.0f} | fc1 dependency-wait exits min {dw.min() - fs:.0f} median {np.median(dw) - fs:.0f} | "
          f"fc1 CTA ends median {np.median(f1[:, 9]) - fs:.0f} max {ce - fs:.0f} | next round starts ~{1000 * per_round:.0f}")
    q = lambda a: " ".join(f"{v:.0f}" for v in np.percentile(a, [0, 10, 25, 50, 75, 90, 100]))
    print(f"   front CTA entries                             : {q(fr[:, 30] - fs)}")
    print(f"   front TMEM allocated                          : {q(fr[:, 29] - fs)}")
    print(f"   front CTA starts (ns, pct 0/10/25/50/75/90/100): {q(fr[:, 13] - fs)}")
    print(f"   front CTA ends                                : {q(fr[:, 14] - fs)}")
    print(f"   fc1 CTA starts                                : {q(f1[:, 8] - fs)}")
    print(f"   fc1 dependency-wait exits                     : {q(f1[:, 12] - fs)}")
    print(f"   fc1 CTA ends                                  : {q(f1[:, 9] - fs)}")
    print(f"   fc1 after TMEM dealloc                        : {q(f1[:, 13] - fs)}")
    print(f"   front after TMEM dealloc                      : {q(fr[:, 31] - fs)}")
    print(f"   next front CTA entries                        : {q(nfr[:, 30] - fs)}")
    print(f"   next front CTA starts                         : {q(nfr[:, 13] - fs)}")
    print(f"   fc1 start->tile0 epilogue: globaltimer {np.median(f1[:, 10] - f1[:, 8]):.0f} ns, clock64 "
          f"{np.median(f1[:, 4] - f1[:, 0]):.0f} cyc; end-start {np.median(f1[:, 9] - f1[:, 8]):.0f} ns")
