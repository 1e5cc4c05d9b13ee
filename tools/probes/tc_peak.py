"""Tensor-core peaks for the roofline (tc_peak.cu): per-MMA issue cost in one
CTA and the dense all-SM throughput of kind::tf32 / f16 / f8f6f4 at
M=128, N=256.  Writes profiles/peaks_tc.json (bench.py's tensor peaks).

  python tools/probes/tc_peak.py [--out profiles/peaks_tc.json]
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "tc_peak.so")
src = os.path.join(here, "tc_peak.cu")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", src, "-o", so])
L = C.CDLL(so)
L.issue_cost.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
L.issue_cost_ts.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
L.issue_cost_warp.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
L.dense_peak.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
MODES = {"tf32": 1, "bf16": 0, "fp8": 3}  # tc_common.cuh kTF32 / kBF16 / kFP8
K = {"tf32": 8, "bf16": 16, "fp8": 32}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default="")
    p.add_argument("--short", action="store_true", help="issue cost from 64 vs 256 MMAs (queue not yet full)")
    p.add_argument("--no-dense", action="store_true")
    a = p.parse_args()
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = np.zeros(2, np.int64)
    res = {"device": torch.cuda.get_device_name(0), "sms": sms, "issue_cycles": {}, "dense_tflops": {}}
    for name, mode in MODES.items():
        for n in (64, 128, 256):
            for nacc in (1, 2, 4):
                if n == 256 and nacc == 4:
                    continue
                r = []
                for count in ((64, 256) if a.short else (256, 1024)):
                    e = L.issue_cost(mode, n, count, nacc, out.ctypes.data)
                    assert e == 0, e
                    r.append((count, int(out[1])))
                per = (r[1][1] - r[0][1]) / (r[1][0] - r[0][0])
                res["issue_cycles"][f"{name}_n{n}_acc{nacc}"] = per
                print(f"{name:5s} M=128 N={n:3d} acc={nacc}: {per:6.1f} cycles/MMA "
                      f"({2 * 128 * n * K[name] / per / 1e3:6.2f} kFLOP/cycle/SM)", flush=True)
    for ts, n, nacc in [(ts, n, nacc) for ts in (0, 1) for n in (64, 128, 256) for nacc in (1, 2)]:
        if True:  # whole-warp issue loop, elect.sync inside the asm; ts: A from tensor memory
            if n == 256 and nacc == 2:
                continue
            r = []
            for count in ((64, 256) if a.short else (256, 1024)):
                e = L.issue_cost_warp(n, count, nacc, out.ctypes.data, ts)
                assert e == 0, e
                r.append((count, int(out[1])))
            per = (r[1][1] - r[0][1]) / (r[1][0] - r[0][0])
            res["issue_cycles"][f"tf32_warp{'_ts' if ts else ''}_n{n}_acc{nacc}"] = per
            print(f"tf32  warp-elect{' A-from-TMEM' if ts else ''} M=128 N={n:3d} acc={nacc}: {per:6.1f} cycles/MMA",
                  flush=True)
    for name in ("tf32", "bf16"):  # A from tensor memory (FC1's form at c3)
        for n in (64, 128, 256):
            for nacc in (1, 2):
                if n == 256 and nacc == 2:
                    continue
                r = []
                for count in ((64, 256) if a.short else (256, 1024)):
                    e = L.issue_cost_ts(MODES[name], n, count, nacc, out.ctypes.data)
                    assert e == 0, e
                    r.append((count, int(out[1])))
                per = (r[1][1] - r[0][1]) / (r[1][0] - r[0][0])
                res["issue_cycles"][f"{name}_ts_n{n}_acc{nacc}"] = per
                print(f"{name:5s} A-from-TMEM M=128 N={n:3d} acc={nacc}: {per:6.1f} cycles/MMA", flush=True)
    for name, mode in MODES.items():
        if a.no_dense:
            break
        tf, ms = C.c_double(), C.c_double()
        e = L.dense_peak(mode, sms, 16384, 1, C.byref(tf), C.byref(ms))  # burst: one launch
        assert e == 0, e
        burst = tf.value
        t0 = time.time()
        vals = []
        while time.time() - t0 < 1.5:  # sustained: back-to-back launches for ~1.5 s
            e = L.dense_peak(mode, sms, 16384, 8, C.byref(tf), C.byref(ms))
            assert e == 0, e
            vals.append(tf.value)
        res["dense_tflops"][name] = {"burst": burst, "sustained": float(np.median(vals[len(vals) // 2:])),
                                     "shape": "M=128 N=256, 2 accumulators, operands in SMEM (SW128)"}
        print(f"{name:5s} dense M=128 N=256: burst {burst:8.1f} TFLOP/s, sustained "
              f"{res['dense_tflops'][name]['sustained']:8.1f} TFLOP/s", flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
