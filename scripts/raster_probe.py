"""Ladder-shape GEMM under several grouped-rasterisation heights (tn_debug_raster), for an ncu
launch list of duration / DRAM bytes / SM clock per setting (exploration only)."""
import ctypes as C
import sys

import numpy as np

from paper_2507_11424_b200 import _lib

LIB = _lib.lib()
LIB.tn_debug_gemm_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
M, N, K = (int(x) for x in sys.argv[1:4])
out = np.zeros(4)
for gm in [int(x) for x in sys.argv[4].split(",")]:
    LIB.tn_debug_raster(gm)
    LIB.tn_debug_gemm_bench(M, N, K, 1, 2, 3, out.ctypes.data)
    print(f"GM={gm}: {out[0]:.3f} ms", flush=True)
