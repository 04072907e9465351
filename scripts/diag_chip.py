"""Diagnostic: per-vertex relative error of the GPU conditionals against the closed form on the
Willow-105 chip-row partition of a K=3 branch superposition (test_chip_row_partition_willow_exact_closed_form)."""
import sys
import numpy as np
from tninputs import lattices as L, synthetic as S
from tests.test_oracle import closed_form_conditionals
from paper_2507_11424_b200 import TNState

lat = L.willow105()
st = S.branch_superposition(lat, 4, 3, seed=5)
st2, rows2, nq = S.split_two_edge_vertices(st, L.chip_rows(lat), [c[0] for c in lat.coords])
u = S.uniforms(6, st2["n"], 19)
order = [v for r in rows2 for v in r if v < nq]
rowof = {v: b for b, r in enumerate(rows2) for v in r}
for opts in [dict(), dict(gemm=1), dict(gemm=2)]:
    for R in (16, 32, 64):
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
                    worst = (e, (k, v, rowof[v], cond[k, v], r))
        print(opts, "R", R, "worst rel", worst, "flags", flags.tolist(), flush=True)
