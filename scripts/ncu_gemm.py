"""One large complex GEMM through the contraction engine (for ncu captures of tc_gemm_kernel)."""
import ctypes as C
import sys

import numpy as np

from paper_2507_11424_b200 import _lib

LIB = _lib.lib()
LIB.tn_debug_gemm_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 4096, 4096)))
out = np.zeros(4)
assert LIB.tn_debug_gemm_bench(M, N, K, 1, 2, 1, out.ctypes.data) == 0
print(f"M={M} N={N} K={K}: {out[0]:.3f} ms, {8.0 * M * N * K / out[0] / 1e9:.1f} TFLOP/s alg, err {out[1]:.2e}")
