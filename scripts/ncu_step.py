"""One sampling step (batch) of a workload inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (precompute and a warm-up batch run outside)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_11424_b200 import TNState  # noqa: E402
from tninputs import lattices as L  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "willow105_chi16_env64"
lat_name, chi, R, batch = bench.WORKLOADS[wl]
if len(sys.argv) > 2:
    batch = int(sys.argv[2])
lat = L.by_name(lat_name)
st = bench.make_state(lat, chi)
g = TNState(st)
g.prepare(lat.rows, R)
g.set_option("max_batch", batch)
u = np.random.default_rng(5).random((batch, lat.n))
g.sample(lat.rows, R, u)
torch.cuda.synchronize()
torch.cuda.profiler.start()
g.sample(lat.rows, R, u)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", wl, batch)
