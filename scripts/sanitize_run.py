"""Small sampling run for compute-sanitizer (memcheck / racecheck / synccheck): every GEMM on the
tcgen05 path (gemm = 2: TMA ring, mbarriers, TMEM, CTA pairs), fits, orthonormalisation,
tail, amplitude; exits non-zero on a mismatch with the exact statevector."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import statevector as SV  # noqa: E402
from paper_2507_11424_b200 import TNState  # noqa: E402
from tninputs import lattices as L  # noqa: E402
from tninputs import synthetic as S  # noqa: E402

lat = L.square(3, 3)
st = S.vidal_like(lat, 2, seed=3, xi=2.0)
g = TNState(st)
g.set_option("gemm", 2)
u = S.uniforms(4, lat.n, 5)
bits, logq, cond, flags = g.sample(lat.rows, 16, u, want_cond=True)
psi = SV.statevector(st)
z = np.vdot(psi, psi).real
for k in range(len(u)):
    lp = math.log(abs(psi[int("".join(map(str, bits[k])), 2)]) ** 2 / z)
    assert abs(logq[k] - lp) < 1e-4 * max(1, abs(lp)), (k, logq[k], lp)
la, ph = g.amplitude(bits, 16)
print("sanitize run ok", g.stats())
