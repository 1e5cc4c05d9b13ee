# diagnostics: row-per-lane vs piece-per-lane 32-B loads (see gather_probe.cu)
import ctypes as C, os, subprocess
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "gather_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                           os.path.join(here, "gather_probe.cu"), "-o", so])
L = C.CDLL(so)
for ctas in (1, 128):
    for mode, name in ((0, "lane = row"), (1, "lanes over pieces")):
        out = np.zeros(ctas, np.int64)
        e = L.probe(ctas, mode, out.ctypes.data_as(C.c_void_p))
        print(f"ctas {ctas:3d} {name:18s}: median {np.median(out):6.0f} cycles (48 KB per CTA), err {e}")
