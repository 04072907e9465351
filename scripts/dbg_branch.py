import math, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2507_11424_b200 import TNState
from tninputs import lattices as L, synthetic as S
from tests.test_oracle import closed_form_conditionals
lat = L.willow105()
st = S.branch_superposition(lat, 32, 4, seed=11)
u = S.uniforms(4, lat.n, 12)
order = [v for r in lat.rows for v in r]
res = {}
for old in ("1", "0"):
    os.environ["TN_ORTH_OLD"] = old
    g = TNState(st)
    bits, logq, cond, flags = g.sample(lat.rows, 16, u, want_cond=True)
    res[old] = (bits, cond, flags)
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k])
        bad = [(i, v, cond[k, v], r) for i, (v, r) in enumerate(zip(order, ref)) if abs(cond[k, v] - r) > 1e-4 * r + 1e-6]
        print("old" if old == "1" else "new", "sample", k, "flags", flags[k], "nbad", len(bad), bad[:3], flush=True)
