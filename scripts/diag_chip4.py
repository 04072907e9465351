"""Exact-regime accuracy vs chi_env on a normalised K=3 branch superposition: chip-row and
plain Willow partitions, both GEMM paths (rank-deficient fits)."""
import numpy as np
from tninputs import lattices as L, synthetic as S
from tests.test_oracle import closed_form_conditionals
from paper_2507_11424_b200 import TNState
lat = L.willow105()
rng = np.random.default_rng(5)
phis = rng.standard_normal((3, lat.n, 2)) + 1j * rng.standard_normal((3, lat.n, 2))
phis /= np.linalg.norm(phis, axis=2, keepdims=True)
st = S.branch_superposition(lat, 4, 3, seed=5, phis=phis)
st2, rows2, nq = S.split_two_edge_vertices(st, L.chip_rows(lat), [c[0] for c in lat.coords])
for name, s, rows, nqq in (("plain", st, lat.rows, lat.n), ("chip", st2, rows2, nq)):
    u = S.uniforms(6, s["n"], 19)
    order = [v for r in rows for v in r if v < nqq]
    for gemm in (0, 1):
        for R in (8, 12, 16, 24, 32, 64):
            g = TNState(s)
            g.set_option("gemm", gemm)
            bits, logq, cond, flags = g.sample(rows, R, u, want_cond=True)
            worst = 0
            for k in range(len(u)):
                ref = closed_form_conditionals(phis, order, bits[k, :nqq])
                worst = max([worst] + [abs(cond[k, v] - r) / r for v, r in zip(order, ref)])
            print(name, "gemm", gemm, "R", R, "worst %.2e" % worst, "lnZ-ln3 %.2e" % (g.log_norm(R) - np.log(3)), flush=True)
