# diagnostics: cycles per back-to-back tcgen05.mma (see mma_probe.cu)
import ctypes as C, os, subprocess
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "mma_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", os.path.join(here, "mma_probe.cu"), "-o", so])
L = C.CDLL(so)
out = np.zeros(2, np.int64)
for mode, name in ((1, "tf32"),):
    for n in (64, 128, 256):
        for ts in (0, 1):
            for nacc in (1, 2, 11, 12):
                if nacc % 10 == 2 and n == 256:
                    continue
                r = []
                for count in (64, 256):
                    e = L.probe(mode, n, count, ts, nacc, out.ctypes.data_as(C.c_void_p))
                    r.append((count, out[0], out[1]))
                (c1, i1, t1), (c2, i2, t2) = r
                per = (t2 - t1) / (c2 - c1)
                print(f"{name} N={n:3d} {'TS' if ts else 'SS'} acc={nacc % 10}{' warp-wide' if nacc > 10 else ''}: {per:6.1f} cyc/MMA (issue {(i2 - i1) / (c2 - c1):5.1f}), "
                      f"floor {128 * n / 256:.0f}; err {e}")

for n in (64, 128):
    for pattern in (0, 1):
        r = []
        for ks in (16, 64):
            e = L.probe_ksteps(n, ks, pattern, out.ctypes.data_as(C.c_void_p))
            r.append((ks, out[1]))
        per = (r[1][1] - r[0][1]) / (r[1][0] - r[0][0])
        print(f"3xTF32 k-step N={n} pattern {'3 MMAs' if pattern == 0 else 'stacked 2N + N'}: {per:6.1f} cyc/k-step; err {e}")
