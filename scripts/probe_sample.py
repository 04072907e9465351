"""One precompute, then time the sampling step at several batch sizes (exploration only).

python scripts/probe_sample.py [workload] [batches...]
"""
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
batches = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
lat_name, chi, R, _ = bench.WORKLOADS[wl]
lat = L.by_name(lat_name)
LIB = _lib.lib()
LIB.tn_debug_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
LIB.tn_debug_set_profile.argtypes = [C.c_int]
LIB.tn_debug_counters.argtypes = [C.c_void_p, C.c_int]
st = bench.make_state(lat, chi)
g = TNState(st)
t0 = time.time()
g.prepare(lat.rows, R)
torch.cuda.synchronize()
print(f"{wl}: precompute {time.time() - t0:.1f} s", flush=True)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
N = lat.n
for nb in batches:
    g.set_option("max_batch", nb)
    T = int(os.environ.get("PROBE_STEPS", "2"))
    u = torch.from_numpy(np.random.default_rng(5).random((2 + T, nb, N))).to(dev)
    bits = torch.empty((2 + T, nb, N), dtype=torch.uint8, device=dev)
    lq = torch.empty((2 + T, nb), dtype=torch.float64, device=dev)

    def step(s):
        g.sample_dev(lat.rows, R, nb, u[s].data_ptr(), bits[s].data_ptr(), lq[s].data_ptr(), 0, 0,
                     stream.cuda_stream)

    step(0)
    step(1)
    torch.cuda.synchronize()
    prof = np.zeros(7)
    LIB.tn_debug_set_profile(1)
    LIB.tn_debug_profile(prof.ctypes.data, None, 7, 1)
    cnt = np.zeros(4)
    LIB.tn_debug_counters(cnt.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s_ in range(2, 2 + T):
        step(s_)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / T
    LIB.tn_debug_profile(prof.ctypes.data, None, 7, 1)
    LIB.tn_debug_set_profile(0)
    LIB.tn_debug_counters(cnt.ctypes.data, 1)
    ph = {k: round(float(v) / T, 1) for k, v in zip(bench.PHASES, prof)}
    print(f"batch {nb}: {ms:.1f} ms/step, {1000 * nb / ms:.3f} samples/s, cMAC/sample {cnt[0] / (T * nb):.3e}; "
          f"phases ms/step {ph}", flush=True)
if os.environ.get("TN_GEMM_LOG"):
    LIB.tn_debug_gemm_log()
    LIB.tn_debug_simt_log()
