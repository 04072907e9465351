import ctypes as C
import numpy as np
from paper_2507_11424_b200 import _lib
LIB = _lib.lib()
LIB.tn_debug_orth_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
out = np.zeros(2)
assert LIB.tn_debug_orth_bench(8192, 128, 2, 1, 0, out.ctypes.data) == 0
print("ok", out[0])
