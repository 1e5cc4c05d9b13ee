# diagnostics: arrival clocks of 4 x 16 KB bulk copies per CTA (see bulk_probe.cu)
import ctypes as C, os, subprocess, sys
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "bulk_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                           os.path.join(here, "bulk_probe.cu"), "-o", so])
L = C.CDLL(so)
for ctas in (32, 128):
    for nch, cb in ((4, 16384), (8, 16384), (2, 32768)):
        for mode, name in ((0, "just written"), (1, "warm (read before)"), (2, "cold (L2 flushed)")):
            out = np.zeros(ctas * 8, np.int64)
            L.probe(ctas, nch, cb, mode, out.ctypes.data_as(C.c_void_p))
            o = out.reshape(ctas, 8)[:, :nch]
            print(f"ctas {ctas:3d} {nch} x {cb // 1024} KB {name:20s}: median arrival cycles " +
                  " ".join(f"{v:6.0f}" for v in np.median(o, 0)))
