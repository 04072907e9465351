"""Time one complex contraction on both GEMM paths (debug entry point, device-resident)."""
import ctypes as C
import os
import sys

import numpy as np

from paper_2507_11424_b200 import _lib

LIB = _lib.lib()
LIB.tn_debug_gemm_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
LIB.tn_debug_last_error.restype = C.c_char_p
shapes = [(32768, 4096, 4096, 2), (16384, 2048, 1024, 4), (8192, 128, 4096, 8), (4096, 4096, 4096, 1),
          (128, 4096, 4096, 4), (300, 2048, 2048, 2), (8192, 16384, 128, 2), (16384, 4096, 128, 2)]
modes = [int(x) for x in os.environ.get("MODES", "2,1").split(",")]
# warm the clocks up (~1-2 s of GEMMs) before timing
out = np.zeros(4)
for _ in range(3):
    LIB.tn_debug_gemm_bench(32768, 4096, 4096, 1, 2, 10, out.ctypes.data)
for M, N, K, nb in shapes:
    for mode in modes:
        if mode == 1 and M * N * K * nb > 2 ** 36:
            continue
        out = np.zeros(4)
        rc = LIB.tn_debug_gemm_bench(M, N, K, nb, mode, int(os.environ.get('REPS', '10')), out.ctypes.data)
        assert rc == 0, LIB.tn_debug_last_error()
        ms, relerr = out[0], out[1]
        tf = 8.0 * M * N * K * nb / (ms * 1e-3) / 1e12
        print(f"M={M} N={N} K={K} nb={nb} mode={mode} tc2={os.environ.get('TN_TC2', '1')}: {ms:.3f} ms  "
              f"{tf:.1f} TFLOP/s (complex-algorithmic, incl. prep)  rel.err vs fp64 sample {relerr:.2e}", flush=True)
