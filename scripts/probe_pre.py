"""Profile the first rows of the norm-environment precompute (TN_PRE_ROWS) at a workload."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_11424_b200 import TNState, _lib  # noqa: E402
from tninputs import lattices as L  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "willow105_chi32_env128"
lat_name, chi, R, _ = bench.WORKLOADS[wl]
lat = L.by_name(lat_name)
LIB = _lib.lib()
LIB.tn_debug_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
LIB.tn_debug_set_profile.argtypes = [C.c_int]
st = bench.make_state(lat, chi)
g = TNState(st)
prof = np.zeros(7)
LIB.tn_debug_set_profile(1)
LIB.tn_debug_profile(prof.ctypes.data, None, 7, 1)
t0 = time.time()
g.prepare(lat.rows, R)
torch.cuda.synchronize()
t = time.time() - t0
LIB.tn_debug_profile(prof.ctypes.data, None, 7, 1)
print(f"{wl}: TN_PRE_ROWS={os.environ.get('TN_PRE_ROWS')} precompute {t:.1f} s; phases (ms)",
      {k: round(float(v), 1) for k, v in zip(bench.PHASES, prof)}, flush=True)
if os.environ.get("TN_GEMM_LOG"):
    LIB.tn_debug_gemm_log()
