"""Dump GPU conditionals on the chip-row partition (normalised branch factors) for offline comparison."""
import numpy as np
from tninputs import lattices as L, synthetic as S
from paper_2507_11424_b200 import TNState
lat = L.willow105()
rng = np.random.default_rng(5)
phis = rng.standard_normal((3, lat.n, 2)) + 1j * rng.standard_normal((3, lat.n, 2))
phis /= np.linalg.norm(phis, axis=2, keepdims=True)
st = S.branch_superposition(lat, 4, 3, seed=5, phis=phis)
st2, rows2, nq = S.split_two_edge_vertices(st, L.chip_rows(lat), [c[0] for c in lat.coords])
u = S.uniforms(6, st2["n"], 19)
out = {}
for tag, R in (("r32", 32), ("r12", 12)):
    g = TNState(st2)
    bits, logq, cond, flags = g.sample(rows2, R, u, want_cond=True)
    out[tag + "_bits"] = bits; out[tag + "_cond"] = cond; out[tag + "_flags"] = flags
    out[tag + "_lnz"] = g.log_norm(R)
np.savez("gpurun_out/chip_gpu_norm.npz", **out)
print("saved", out["r32_lnz"], out["r12_lnz"])
