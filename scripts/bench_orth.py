"""Time batched orthonormalisation (debug entry point) at the fit's panel shapes."""
import ctypes as C
import os

import numpy as np

from paper_2507_11424_b200 import _lib

LIB = _lib.lib()
LIB.tn_debug_orth_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
for m, n, nb in [(8192, 128, 2), (8192, 128, 1), (4096, 128, 2), (1024, 64, 16), (2048, 32, 16)]:
    out = np.zeros(2)
    assert LIB.tn_debug_orth_bench(m, n, nb, 20, 0, out.ctypes.data) == 0
    print(f"orth m={m} n={n} nb={nb} old={os.environ.get('TN_ORTH_OLD', '0')}: {out[0]:.3f} ms", flush=True)
LIB.tn_debug_chol_clocks.argtypes = [C.c_void_p]
clk = np.zeros(3, dtype=np.int64)
LIB.tn_debug_orth_bench(8192, 128, 1, 1, 0, np.zeros(2).ctypes.data)
LIB.tn_debug_chol_clocks(clk.ctypes.data)
print("chol clocks (load, factor, inverse) of the last call:", clk.tolist())
LIB.tn_debug_chol_flags.argtypes = [C.c_int]
LIB.tn_debug_chol_flags(1)
LIB.tn_debug_orth_bench(8192, 128, 1, 1, 0, np.zeros(2).ctypes.data)
LIB.tn_debug_chol_clocks(clk.ctypes.data)
print("chol clocks without the Schur update:", clk.tolist())
LIB.tn_debug_chol_flags(0)
