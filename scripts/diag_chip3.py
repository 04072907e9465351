import os, sys
import numpy as np
from tninputs import lattices as L, synthetic as S
from tests.test_oracle import closed_form_conditionals
from paper_2507_11424_b200 import TNState
lat = L.willow105()
st = S.branch_superposition(lat, 4, 3, seed=5)
st2, rows2, nq = S.split_two_edge_vertices(st, L.chip_rows(lat), [c[0] for c in lat.coords])
u = S.uniforms(3, st2["n"], 19)
order = [v for r in rows2 for v in r if v < nq]
rowof = {v: b for b, r in enumerate(rows2) for v in r}
tag = sys.argv[1]
for opts in [dict(), dict(fit_half_sweeps=4), dict(fit_half_sweeps=6), dict(init_seed=7), dict(order=1)]:
    for R in (12, 32):
        g = TNState(st2)
        for k, v in opts.items():
            g.set_option(k, v)
        bits, logq, cond, flags = g.sample(rows2, R, u, want_cond=True)
        worst = (0, None)
        for k in range(len(u)):
            ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k, :nq])
            for v, r in zip(order, ref):
                e = abs(cond[k, v] - r) / r
                if e > worst[0]:
                    worst = (e, (k, v, rowof[v]))
        print(tag, opts, "R", R, "worst rel %.3e" % worst[0], worst[1], "lnZ", g.log_norm(R), flush=True)
