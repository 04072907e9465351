"""Host enqueue time vs device time of sampling steps (is the step launch-bound?)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2507_11424_b200 import TNState  # noqa: E402
from tninputs import lattices as L  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "willow105_chi32_env128"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lat_name, chi, R, _ = bench.WORKLOADS[wl]
lat = L.by_name(lat_name)
g = TNState(bench.make_state(lat, chi))
if os.environ.get("RASTER_GM"):
    from paper_2507_11424_b200 import _lib
    _lib.lib().tn_debug_raster(int(os.environ["RASTER_GM"]))
g.prepare(lat.rows, R)
g.set_option("max_batch", nb)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
N = lat.n
u = torch.from_numpy(np.random.default_rng(5).random((8, nb, N))).to(dev)
bits = torch.empty((8, nb, N), dtype=torch.uint8, device=dev)
lq = torch.empty((8, nb), dtype=torch.float64, device=dev)


def step(s):
    g.sample_dev(lat.rows, R, nb, u[s].data_ptr(), bits[s].data_ptr(), lq[s].data_ptr(), 0, 0, stream.cuda_stream)


for s in range(2):
    step(s)
torch.cuda.synchronize()
for s in range(2, 6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    t0 = time.perf_counter()
    step(s)
    th = time.perf_counter() - t0
    e1.record(stream)
    torch.cuda.synchronize()
    tw = time.perf_counter() - t0
    print(f"step {s}: host enqueue {1e3 * th:.1f} ms, wall {1e3 * tw:.1f} ms, device {e0.elapsed_time(e1):.1f} ms",
          flush=True)
