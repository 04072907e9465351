"""Time the GPU TNS construction (NEXT-4) of the domain-wall quench on Willow-105."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11424_b200 import construct  # noqa: E402
from tninputs import lattices as L  # noqa: E402

torch.cuda.set_device(0)
lat = L.willow105()
for chi, layers in [(int(a.split(":")[0]), int(a.split(":")[1])) for a in sys.argv[1:]]:
    t0 = time.time()
    st = construct.heisenberg_quench(lat, L.domain_wall_bits(lat), chi, layers)
    print(f"willow105 chi={chi} L={layers}: {time.time() - t0:.1f} s, fidelity {st['meta']['fidelity']:.5f}, "
          f"max bond {max(st['bond_dims'])}, gates {len(st['meta']['eps'])}, BP residual max "
          f"{st['meta']['bp_residual_max']:.2e}", flush=True)
