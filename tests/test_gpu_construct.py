"""NEXT-4: TNS construction on the GPU (libtnsample tn_su_*: FP64 BP +
BP-gauged simple update) against the oracle generator (oracle/generator.py, O7) on the same
circuits: the same represented state (statevector overlap, or the same sampling distribution
through the GPU sampler), the same discarded weights eps_i (Eq. 1) and bond
dimensions. Bases differ by gauges on the bonds (R7), so tensors are not compared directly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import generator as G  # noqa: E402
from oracle import statevector as SV  # noqa: E402
from paper_2507_11424_b200 import TNState  # noqa: E402
from paper_2507_11424_b200 import construct as CG  # noqa: E402
from tninputs import lattices as L  # noqa: E402
from tninputs import synthetic as S  # noqa: E402


def _overlap(a, b):
    return abs(np.vdot(a, b)) / (np.linalg.norm(a) * np.linalg.norm(b))


def test_gate_closed_forms_match_oracle():
    for th in (0.1, 0.37, -1.2):
        assert np.allclose(CG.heisenberg_gate(1.0, th), G.heisenberg_gate(1.0, th), atol=1e-15)
        assert np.allclose(CG.xxpyy_gate(th), G.xxpyy_gate(th), atol=1e-15)
        assert np.allclose(CG.cphase_gate(th), G.cphase_gate(th), atol=1e-15)


def test_su_untruncated_is_the_oracle_state():
    """without truncation the TNS is exact -- the GPU-built state equals the oracle
    generator's (statevector overlap 1 to 1e-10), every eps_i ~ 0."""
    lat = L.square(2, 3)
    bits = L.domain_wall_bits(lat)
    ref = G.heisenberg_quench(lat, chi=64, layers=3)
    got = CG.heisenberg_quench(lat, bits, chi=64, layers=3)
    assert _overlap(SV.statevector(got), SV.statevector(ref)) > 1 - 1e-10
    assert max(got["meta"]["eps"]) < 1e-12
    assert list(got["bond_dims"]) == list(ref["bond_dims"])


@pytest.mark.parametrize("name,lat_name,chi,layers", [("cfg1", "square3x3", 4, 2), ("sq34", "square3x4", 3, 3)])
def test_su_truncated_matches_oracle(name, lat_name, chi, layers):
    """Truncating simple update (config 1 and a 3x4 lattice at chi = 3): the same eps_i sequence
    (Eq. 1), the same bond dimensions and the same represented state as the oracle generator."""
    lat = L.by_name(lat_name)
    bits = L.domain_wall_bits(lat)
    ref = G.heisenberg_quench(lat, chi=chi, layers=layers)
    got = CG.heisenberg_quench(lat, bits, chi=chi, layers=layers)
    assert list(got["bond_dims"]) == list(ref["bond_dims"])
    e1, e2 = np.asarray(got["meta"]["eps"]), np.asarray(ref["meta"]["eps"])
    assert len(e1) == len(e2)
    assert np.allclose(e1, e2, rtol=1e-6, atol=1e-10), np.abs(e1 - e2).max()
    assert abs(got["meta"]["fidelity"] - ref["meta"]["fidelity"]) < 1e-8
    assert _overlap(SV.statevector(got), SV.statevector(ref)) > 1 - 1e-8


def test_su_willow_state_samples_like_the_oracle_state():
    """Full Willow-105 topology, 2 Trotter layers at chi = 4 (truncating): the GPU-built and the
    oracle-built states give the same conditionals under the GPU sampler (chi_env = 16, R16)."""
    lat = L.willow105()
    bits = L.domain_wall_bits(lat)
    ref = G.heisenberg_quench(lat, chi=4, layers=2)
    got = CG.heisenberg_quench(lat, bits, chi=4, layers=2)
    assert list(got["bond_dims"]) == list(ref["bond_dims"])
    assert np.allclose(got["meta"]["eps"], ref["meta"]["eps"], rtol=1e-5, atol=1e-10)
    u = S.uniforms(8, lat.n, 5)
    b1, l1, c1, _ = TNState(got).sample(lat.rows, 16, u, want_cond=True)
    b2, l2, c2, _ = TNState(ref).sample(lat.rows, 16, u, want_cond=True)
    same = (b1 == b2).all(axis=1)
    assert same.mean() >= 0.75
    assert np.allclose(l1[same], l2[same], rtol=1e-4, atol=1e-4)
