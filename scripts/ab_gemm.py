"""A/B timing of two builds of libtnsample.so in one process (alternating calls, same clocks).

python scripts/ab_gemm.py old.so new.so  -- per shape: median ms of the contraction (prep + kernel)
"""
import ctypes as C
import sys

import numpy as np

libs = []
for path in sys.argv[1:3]:
    lib = C.CDLL(path)
    lib.tn_debug_gemm_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    libs.append(lib)
shapes = [(32768, 4096, 4096, 1), (16384, 128, 4096, 4), (8192, 16384, 128, 4), (16384, 2048, 1024, 4),
          (65536, 1024, 2048, 1)]
out = np.zeros(4)
for lib in libs:  # warm up
    lib.tn_debug_gemm_bench(32768, 4096, 4096, 1, 2, 5, out.ctypes.data)
for M, N, K, nb in shapes:
    t = [[], []]
    for rep in range(5):
        for i, lib in enumerate(libs):
            assert lib.tn_debug_gemm_bench(M, N, K, nb, 2, 3, out.ctypes.data) == 0
            t[i].append(out[0])
    a, b = np.median(t[0]), np.median(t[1])
    print(f"M={M} N={N} K={K} nb={nb}: old {a:.3f} ms  new {b:.3f} ms  new/old {b / a:.3f}  err old {out[1]:.1e}",
          flush=True)
