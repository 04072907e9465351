"""Input generators (tninputs): lattice structure and the synthetic states' construction."""
import itertools

import numpy as np
import pytest

from tninputs import lattices as L
from tninputs import synthetic as S


def _check_colouring(lat):
    seen = sorted(e for g in lat.colours for e in g)
    assert seen == list(range(lat.n_edges))
    for g in lat.colours:  # each group is a matching ("each site at most once")
        vs = [v for e in g for v in lat.edges[e]]
        assert len(vs) == len(set(vs))


@pytest.mark.parametrize("name,n,ne,loops,widths", [
    ("willow105", 105, 182, 78, [1, 3, 5, 7, 9, 11, 13, 14, 12, 10, 8, 6, 4, 2]),
    ("eagle127", 127, 144, 18, [14, 4, 15, 4, 15, 4, 15, 4, 15, 4, 15, 4, 14]),
    ("lucj52", 52, 57, 6, [2] * 26),
    ("lucj72", 72, 75, 4, [2] * 36),
    ("square3x3", 9, 12, 4, [3] * 3),
    ("square6x6", 36, 60, 25, [6] * 6),
])
def test_lattice_counts(name, n, ne, loops, widths):
    lat = L.by_name(name)
    assert (lat.n, lat.n_edges, lat.n_loops()) == (n, ne, loops)
    assert [len(r) for r in lat.rows] == widths
    _check_colouring(lat)
    # minimum K equals the coordination number z on bipartite lattices
    assert len(lat.colours) == max(lat.degree())


def test_lucj_loops_match_paper():
    # "sublattices ... with 6 and 4 primitive loops"
    assert L.by_name("lucj52").n_loops() == 6
    assert L.by_name("lucj72").n_loops() == 4


def test_domain_wall_halves():
    for name in ("willow105", "eagle127", "square6x6"):
        lat = L.by_name(name)
        bits = L.domain_wall_bits(lat)
        assert sum(bits) == lat.n - lat.n // 2


def _dense(st):
    from oracle.statevector import statevector  # oracle is test infrastructure
    return statevector(st)


def test_branch_superposition_is_branch_sum():
    lat = L.square(2, 3)
    st = S.branch_superposition(lat, 4, 3, seed=5)
    psi = _dense(st)
    phis = st["meta"]["phis"]
    ref = np.zeros(2 ** lat.n, dtype=complex)
    for idx, x in enumerate(itertools.product([0, 1], repeat=lat.n)):
        ref[idx] = sum(np.prod([phis[c, v, x[v]] for v in range(lat.n)]) for c in range(3))
    assert np.allclose(psi, ref, atol=1e-10 * np.abs(ref).max())


def test_ghz_and_product():
    lat = L.square(2, 2)
    psi = _dense(S.ghz(lat, chi=3, seed=1))
    ref = np.zeros(16, dtype=complex)
    ref[0] = ref[15] = 1
    assert np.allclose(psi, ref, atol=1e-10)
    psi = _dense(S.product_state(lat, [0, 1, 1, 0]))
    assert abs(psi[0b0110]) == 1 and np.count_nonzero(psi) == 1


def test_relabel_preserves_state():
    lat = L.square(2, 3)
    st = S.vidal_like(lat, 2, seed=2)
    perm = [3, 0, 5, 1, 4, 2]
    st2, rows2 = S.relabel(st, lat.rows, perm)
    psi = _dense(st).reshape([2] * 6)
    psi2 = _dense(st2).reshape([2] * 6)
    # vertex v of st is vertex perm[v] of st2
    assert np.allclose(np.transpose(psi2, perm), psi)
    assert sorted(v for r in rows2 for v in r) == list(range(6))


def test_uniforms_reproducible():
    a = S.uniforms(4, 7, 11)
    b = np.random.default_rng(11).random((4, 7))
    assert np.array_equal(a, b) and a.min() >= 0 and a.max() < 1
