"""Timing probe: prepare (norm environments) + sampling on synthetic Vidal-like states."""
import argparse
import os
import time

import numpy as np
import torch

from paper_2507_11424_b200 import TNState
from tninputs import lattices as L
from tninputs import synthetic as S

ap = argparse.ArgumentParser()
ap.add_argument("--lat", default="willow105")
ap.add_argument("--chi", type=int, default=8)
ap.add_argument("--R", type=int, default=32)
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--gemm", type=int, default=0)
ap.add_argument("--max_batch", type=int, default=0)
ap.add_argument("--skip_sample", action="store_true")
a = ap.parse_args()

lat = L.by_name(a.lat)
t0 = time.time()
st = S.vidal_like(lat, a.chi, seed=1)
print(f"state gen {time.time() - t0:.1f}s", flush=True)
g = TNState(st)
g.set_option("gemm", a.gemm)
if a.max_batch:
    g.set_option("max_batch", a.max_batch)
t0 = time.time()
g.prepare(lat.rows, a.R)
torch.cuda.synchronize()
print(f"prepare {time.time() - t0:.2f}s stats {g.stats()}", flush=True)
if not a.skip_sample:
    u = S.uniforms(a.n, lat.n, 3)
    g.sample(lat.rows, a.R, u[: min(4, a.n)])
    t0 = time.time()
    bits, logq, cond, flags = g.sample(lat.rows, a.R, u)
    dt = time.time() - t0
    print(f"sample n={a.n} {dt:.3f}s -> {a.n / dt:.1f} samples/s; stats {g.stats()}; flags {np.bincount(flags)}",
          flush=True)

try:
    import ctypes as C
    from paper_2507_11424_b200 import _lib
    LIB = _lib.lib()
    ms = np.zeros(6)
    cnt = np.zeros(6, dtype=np.int64)
    on = LIB.tn_debug_profile(ms.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p), 6, 1)
    if on:
        names = ["gemm_tc", "gemm_simt", "permute", "orth", "tail", "misc"]
        print("profile (ms, count, all calls in this process):",
              {n: (round(m, 1), int(k)) for n, m, k in zip(names, ms, cnt)})
except Exception as e:  # noqa
    print("no profile:", e)
if os.environ.get("TN_GEMM_LOG"):
    LIB.tn_debug_gemm_log()
