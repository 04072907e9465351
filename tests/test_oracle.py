"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Every oracle function is pinned here by something other than itself: the brute-force
statevector (exact regime, "Equality is only achieved if R_x and R_n are large
enough"), closed forms (branch superpositions, GHZ, product states), a published test
vector (SplitMix64), worked examples (Eq. 1, KLD), physical invariants (U(1))
and gauge invariance of the one-site fit (R7).
"""
import itertools
import math
import os

import numpy as np
import pytest
import scipy.linalg

from oracle import bmps as B
from oracle import generator as G
from oracle import statevector as SV
from tninputs import lattices as L
from tninputs import synthetic as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def order_of(rows):
    return [v for r in rows for v in r]


def closed_form_conditionals(phis, order, bits):
    """P(x_v | earlier) for |psi> = sum_c prod_v phi_v^(c) (maths, not the method):
    sum over the free vertices of |amp|^2 factorises into <phi_v^(c')|phi_v^(c)>."""
    K = phis.shape[0]
    n = phis.shape[1]
    gram = np.einsum("cvs,dvs->vcd", phis, phis.conj())  # [v, c, c'] = <phi^c'|phi^c>

    def marg(fixed):
        tot = 0
        for c in range(K):
            for d in range(K):
                t = 1
                for v in range(n):
                    if v in fixed:
                        t *= phis[c, v, fixed[v]] * np.conj(phis[d, v, fixed[v]])
                    else:
                        t *= gram[v, c, d]
                tot += t
        return tot.real

    out, fixed = [], {}
    prev = marg(fixed)
    for v in order:
        fixed[v] = bits[v]
        cur = marg(fixed)
        out.append(cur / prev)
        prev = cur
    return out


# ------------------------------------------------------------------ golden / arithmetic
def test_splitmix64_published_vector():
    vals = [int(x) for x in open(os.path.join(GOLDEN, "splitmix64_1234567.txt"))
            if x.strip() and not x.startswith("#")]
    seed, outs = vals[0], vals[1:]
    state = seed
    for want in outs:
        assert B.splitmix64(state) == want
        state = (state + 0x9E3779B97F4A7C15) % 2 ** 64


def test_hash_init_vectorised_matches_scalar():
    o = B.hash_init((3, 2, 2), B.DEFAULT_SEED, B.TAG_N, 4, 2)
    base = ((((B.DEFAULT_SEED * 31 + 1) * 1000003 + 4) * 1000003 + 2) * 4294967311) % 2 ** 64
    for i in range(12):
        re = (B.splitmix64((base + 2 * i) % 2 ** 64) >> 40) * 2.0 ** -23 - 1
        im = (B.splitmix64((base + 2 * i + 1) % 2 ** 64) >> 40) * 2.0 ** -23 - 1
        assert o.reshape(-1)[i] == complex(re, im)
    assert np.all(np.abs(o.real) <= 1) and np.all(o.real.astype(np.float32) == o.real)


def test_eq1_worked_example():
    """Eq. (1) through the generator's own truncation (generator.apply2):
    on a 4-qubit chain, Bell pairs on (0,1) and (2,3) and the operator
    G = sum_k sqrt(w_k) P_k (x) P_k (P = I, X, Y, Z / sqrt 2) on the middle edge make the
    (01|23) Schmidt spectrum equal the worked example's {0.8, 0.15, 0.04, 0.01} (the Choi state
    of G); truncating the middle bond to chi = 2 must record eps = 0.05."""
    line = [l for l in open(os.path.join(GOLDEN, "eq1_discarded_weight.txt")) if not l.startswith("#")][0]
    spec, keep, want = line.split(";")
    w = np.array([float(x) for x in spec.split()])
    I2 = np.eye(2)
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    Y = np.array([[0, -1j], [1j, 0]])
    Z = np.diag([1.0, -1.0]).astype(complex)
    Gop = sum(np.sqrt(wk) * np.kron(Pk, Pk) / 2 for wk, Pk in zip(w, (I2, X, Y, Z)))
    H = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    CNOT = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    bell = CNOT @ np.kron(H, I2)  # |00> -> (|00> + |11>)/sqrt 2, index 2 x_u + x_v
    lat = L.chain(4)
    tns = G.TNS(lat, [0, 0, 0, 0])
    tns.bp()
    tns.apply2(0, bell, 4)
    tns.apply2(2, bell, 4)
    assert tns.eps[-2:] == [0.0, 0.0]
    tns.bp()
    tns.apply2(1, Gop, int(keep))
    assert abs(tns.eps[-1] - float(want)) < 1e-12, tns.eps[-1]


def test_norm_estimate_pins():
    """E_q[p/q] = <psi|psi> by oracle.metrics.norm_estimate.
    (a) Worked example (tests/golden/norm_estimate_worked.txt): ratios {1, 2, 3, 4} ->
    mean 2.5, standard error sqrt(5/3)/2. (b) Exact regime (config-1-like 3x3
    state scaled so <psi|psi> != 1): q = p/<psi|psi> for every sample, so the estimate is
    <psi|psi> of the brute-force statevector with zero spread."""
    from oracle import metrics
    rows = [l.split() for l in open(os.path.join(GOLDEN, "norm_estimate_worked.txt"))
            if l.strip() and not l.startswith("#")]
    ratios = [float(x) for x in rows[0]]
    want_mean, want_se = float(rows[1][0]), float(rows[1][1])
    m, se = metrics.norm_estimate(np.zeros(len(ratios)), np.log(ratios))
    assert abs(m - want_mean) < 1e-15 and abs(se - want_se) < 1e-12
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    st["tensors"] = [t * 1.3 for t in st["tensors"]]
    psi = SV.statevector(st)
    Z = np.vdot(psi, psi).real
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 16)
    u = S.uniforms(12, lat.n, 5)
    logq, logp = [], []
    for k in range(len(u)):
        bits, lq, _, _ = B.sample(P, M, 16, u[k])
        logq.append(lq)
        logp.append(math.log(abs(psi[int("".join(map(str, bits)), 2)]) ** 2))
    m, se = metrics.norm_estimate(logq, logp)
    assert abs(m / Z - 1) < 1e-10 and se < 1e-10 * Z


def test_importance_expectation_product_state():
    """PAPER.md:297-300, observable Z_i (not the identity): samples = all 2^N basis states with
    uniform q, p = |<x|psi>|^2 of a product state prod_v (a_v|0> + b_v|1>); the importance
    estimate of <Z_i> must equal the closed form (|a_i|^2 - |b_i|^2) / (|a_i|^2 + |b_i|^2)."""
    from oracle import metrics
    rng = np.random.default_rng(4)
    n = 5
    ab = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
    xs = np.array(list(itertools.product([0, 1], repeat=n)))
    amp = np.array([np.prod([ab[v, x[v]] for v in range(n)]) for x in xs])
    logp = np.log(np.abs(amp) ** 2)
    logq = np.full(len(xs), -n * math.log(2))
    for i in range(n):
        zi = 1 - 2 * xs[:, i]
        want = (abs(ab[i, 0]) ** 2 - abs(ab[i, 1]) ** 2) / (abs(ab[i, 0]) ** 2 + abs(ab[i, 1]) ** 2)
        assert abs(metrics.importance_expectation(logq, logp, zi) - want) < 1e-12


def test_heisenberg_gate_closed_form():
    X = np.array([[0, 1], [1, 0]])
    Y = np.array([[0, -1j], [1j, 0]])
    Z = np.diag([1, -1])
    H = np.kron(X, X) + np.kron(Y, Y) + np.kron(Z, Z)
    for J, dt in ((1.0, 0.1), (0.7, 0.3)):
        assert np.allclose(G.heisenberg_gate(J, dt), scipy.linalg.expm(-1j * J * dt * H), atol=1e-14)
    # XX+YY(theta) = exp(-i theta/4 (XX+YY))
    for th in (0.3, -1.1):
        assert np.allclose(G.xxpyy_gate(th), scipy.linalg.expm(-1j * th / 4 * (np.kron(X, X) + np.kron(Y, Y))))


# ------------------------------------------------------------------ generator
def _exact_circuit(lat, layers, J=1.0, dt=0.1):
    n = lat.n
    bits0 = L.domain_wall_bits(lat)
    vec = np.zeros(2 ** n, complex)
    vec[int("".join(map(str, bits0)), 2)] = 1
    g = G.heisenberg_gate(J, dt)
    for _ in range(layers):
        for grp in lat.colours:
            for e in grp:
                u, v = lat.edges[e]
                T = np.moveaxis(vec.reshape([2] * n), [u, v], [0, 1])
                sh = T.shape
                T = (g @ T.reshape(4, -1)).reshape(sh)
                vec = np.moveaxis(T, [0, 1], [u, v]).reshape(-1)
    return vec


def test_generator_untruncated_is_exact():
    """'when the bond dimension is not truncated ... the tensor network is an
    exact representation' -> f = 1 and amplitudes equal the circuit statevector."""
    lat = L.square(2, 3)
    st = G.heisenberg_quench(lat, chi=64, layers=3)
    assert abs(st["meta"]["fidelity"] - 1) < 1e-12
    psi = SV.statevector(st)
    ref = _exact_circuit(lat, 3)
    ov = abs(np.vdot(ref, psi)) / np.linalg.norm(psi)
    # message pseudo-inverses are regularised at 1e-12 (R20/S:81), so 'exact' holds to ~1e-9
    assert abs(ov - 1) < 1e-8


def test_generator_tree_single_truncation():
    """Eq. (1) is exact without loops: on a chain, eps_i = 1 - |<psi_i|G|psi>|^2."""
    lat = L.chain(4)
    st = G.heisenberg_quench(lat, chi=8, layers=2, dt=0.4)
    psi0 = SV.statevector(st)
    psi0 /= np.linalg.norm(psi0)
    tns = G.TNS(lat, [0, 1, 0, 1])
    tns.t = [t.copy() for t in st["tensors"]]
    tns.dims = [int(d) for d in st["bond_dims"]]
    tns.bp()
    g = G.heisenberg_gate(1.0, 0.9)
    tns.apply2(1, g, 1)  # truncate the middle bond to 1
    psi1 = SV.statevector(tns.state(1, {}))
    psi1 /= np.linalg.norm(psi1)
    T = np.moveaxis(psi0.reshape([2] * 4), [1, 2], [0, 1])
    sh = T.shape
    exact = np.moveaxis((g @ T.reshape(4, -1)).reshape(sh), [0, 1], [1, 2]).reshape(-1)
    fid = abs(np.vdot(psi1, exact)) ** 2
    assert abs(tns.eps[-1] - (1 - fid)) < 1e-10


def test_generator_conserves_magnetisation():
    """the Heisenberg gates are U(1) -> every basis state with weight has the
    domain wall's number of ones."""
    lat = L.square(3, 3)
    st = G.heisenberg_quench(lat, chi=4, layers=2)
    psi = SV.statevector(st)
    ones = sum(L.domain_wall_bits(lat))
    w = np.abs(psi) ** 2
    for idx in np.nonzero(w > 1e-20 * w.max())[0]:
        assert bin(int(idx)).count("1") == ones


# ------------------------------------------------------------------ boundary MPS fit
def _random_strip(rng, W=4, chi=3, mu=2, p=2):
    tops, mats = [], []
    for j in range(W):
        l = 1 if j == 0 else chi
        r = 1 if j == W - 1 else chi
        ml = 1 if j == 0 else mu
        mr = 1 if j == W - 1 else mu
        tops.append(rng.standard_normal((ml, 2, mr)) + 1j * rng.standard_normal((ml, 2, mr)))
        mats.append(rng.standard_normal((2, p, l, r)) + 1j * rng.standard_normal((2, p, l, r)))
    return B.Strip("single", tops, mats, [True] * W)


def _dense_strip(strip):
    T = np.ones((1, 1, 1), dtype=complex)  # [phys..., m bond, row bond]
    T = T.reshape(1, 1)
    acc = np.ones((1, 1, 1))  # [P, m, r]
    for j in range(strip.W):
        X = np.einsum("Pmy,mun->Pynu", acc, strip.tops[j])
        X = np.einsum("Pynu,upyr->Ppnr", X, strip.mats[j])
        acc = X.reshape(-1, X.shape[2], X.shape[3])
    return acc.reshape(-1)


def _dense_mps(sites):
    v = np.ones((1, 1))
    for s in sites:
        v = np.einsum("Pa,apb->Ppb", v, s).reshape(-1, s.shape[-1])
    return v.reshape(-1)


def test_fit_exact_when_bond_suffices():
    """O3: with D_k >= rank_k(T) the one-site fit reproduces the dense strip contraction."""
    rng = np.random.default_rng(7)
    strip = _random_strip(rng)
    T = _dense_strip(strip)
    sites, lg = B.fit(strip, R=64, tag=1, b1=1)
    out = _dense_mps(sites) * math.exp(lg)
    assert np.allclose(out, T, atol=1e-10 * np.abs(T).max())


def test_fit_truncated_is_basis_independent(monkeypatch):
    """R7: at finite R the fitted state depends only on the spans, not on the orthonormal
    basis chosen by the QR."""
    rng = np.random.default_rng(8)
    strip = _random_strip(rng, W=5, chi=3, mu=3)
    s1, l1 = B.fit(strip, R=3, tag=1, b1=2)
    ref = _dense_mps(s1) * math.exp(l1)
    rot = np.random.default_rng(9)
    lo, ro = B.left_orth, B.right_orth

    def left(o):
        q = lo(o)
        d = q.shape[-1]
        U, _ = np.linalg.qr(rot.standard_normal((d, d)) + 1j * rot.standard_normal((d, d)))
        return np.tensordot(q, U, axes=([q.ndim - 1], [0]))

    def right(o):
        q, l = ro(o)
        d = q.shape[0]
        U, _ = np.linalg.qr(rot.standard_normal((d, d)) + 1j * rot.standard_normal((d, d)))
        return np.tensordot(U, q, axes=([1], [0])), l @ U.conj().T

    monkeypatch.setattr(B, "left_orth", left)
    monkeypatch.setattr(B, "right_orth", right)
    s2, l2 = B.fit(strip, R=3, tag=1, b1=2)
    out = _dense_mps(s2) * math.exp(l2)
    assert np.allclose(out, ref, atol=1e-10 * np.abs(ref).max())
    T = _dense_strip(strip)
    assert np.linalg.norm(out - T) > 1e-3 * np.linalg.norm(T)  # really truncated


# ------------------------------------------------------------------ sampler, exact regime
def _all_q(P, M, R, n):
    qs = {}
    for x in itertools.product([0, 1], repeat=n):
        bits, logq, cond, _ = B.sample(P, M, R, np.zeros(n), forced=np.array(x))
        qs[x] = math.exp(logq)
    return qs


def test_config1_exact_distribution():
    """config 1 (3x3, chi=4, chi_env=16) is exact under R6, so q(x) equals the
    statevector distribution for all 512 x and sums to 1."""
    lat, st = G.config_state("cfg1")
    psi = SV.statevector(st)
    p = np.abs(psi) ** 2 / np.vdot(psi, psi).real
    P = B.Prepared(st, lat.rows)
    M, logs = B.norm_envs(P, 16)
    assert abs(B.log_norm(P, M, logs) - math.log(np.vdot(psi, psi).real)) < 1e-10
    qs = _all_q(P, M, 16, lat.n)
    assert abs(sum(qs.values()) - 1) < 1e-12
    for x, q in qs.items():
        idx = int("".join(map(str, x)), 2)
        assert abs(q - p[idx]) < 1e-12
    # drawn samples: conditionals equal the statevector conditionals
    u = S.uniforms(16, lat.n, 1001)
    for k in range(16):
        bits, logq, cond, fl = B.sample(P, M, 16, u[k])
        ref = SV.conditionals(psi, lat.n, order_of(lat.rows), bits)
        assert np.allclose([cond[v] for v in order_of(lat.rows)], ref, rtol=1e-10)
        assert fl & 2 == 0  # bit0 may flag a -1e-17 clamp of a U(1)-forbidden branch
        assert sum(bits) == sum(L.domain_wall_bits(lat))  # U(1)


def test_chi_square_config1():
    """Drawn samples follow q = p (chi-square at alpha = 0.001, SPEC.md:500 / S:604),
    with 3000 samples on the 126-state sector to keep the CPU suite short."""
    lat, st = G.config_state("cfg1")
    psi = SV.statevector(st)
    p = np.abs(psi) ** 2 / np.vdot(psi, psi).real
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 16)
    n = 3000
    u = S.uniforms(n, lat.n, 1001)
    counts = {}
    for k in range(n):
        bits, *_ = B.sample(P, M, 16, u[k])
        idx = int("".join(map(str, bits)), 2)
        counts[idx] = counts.get(idx, 0) + 1
    idxs = [i for i in range(512) if p[i] * n >= 5]
    rest = 1 - sum(p[i] for i in idxs)
    obs = [counts.get(i, 0) for i in idxs] + [n - sum(counts.get(i, 0) for i in idxs)]
    exp = [p[i] * n for i in idxs] + [rest * n]
    if exp[-1] < 1e-9:
        obs, exp = obs[:-1], exp[:-1]
    chi2 = sum((o - e) ** 2 / e for o, e in zip(obs, exp))
    assert scipy.stats.chi2.sf(chi2, len(obs) - 1) > 1e-3


@pytest.mark.parametrize("lat_name,chi,K,R,seed", [
    ("square4x4", 4, 3, 16, 1),
    ("willow105", 4, 2, 8, 2),
])
def test_branch_superposition_closed_form(lat_name, chi, K, R, seed):
    """Full-topology pin: rank <= K (single layer) and <= K^2 (double layer) <= R makes the
    method exact, so the conditionals equal the closed form of the branch sum."""
    import scipy  # noqa: F401
    lat = L.by_name(lat_name)
    st = S.branch_superposition(lat, chi, K, seed)
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, R)
    u = S.uniforms(3, lat.n, 77)
    order = order_of(lat.rows)
    for k in range(3):
        bits, logq, cond, fl = B.sample(P, M, R, u[k])
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits)
        assert np.allclose([cond[v] for v in order], ref, rtol=1e-8, atol=1e-12)
        assert abs(logq - sum(math.log(r) for r in ref)) < 1e-8 * max(1, abs(logq))


def test_ghz_eagle_full_scale():
    """S:460 / SURVEY 8(c.4): GHZ on Eagle-127 -> all bits equal, q = 1/2."""
    lat = L.eagle127()
    st = S.ghz(lat, chi=2)
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 4)
    u = S.uniforms(2, lat.n, 3)
    for k in range(2):
        bits, logq, cond, fl = B.sample(P, M, 4, u[k])
        assert len(set(bits.tolist())) == 1
        assert abs(logq - math.log(0.5)) < 1e-10


def test_product_state_reproduces_bits():
    """a product state yields its own bitstring with q = p = 1."""
    lat = L.square(3, 4)
    want = [1, 0, 0, 1, 1, 1, 0, 0, 1, 0, 1, 0]
    st = S.product_state(lat, want)
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 4)
    bits, logq, cond, fl = B.sample(P, M, 4, S.uniforms(1, lat.n, 0)[0])
    assert bits.tolist() == want and logq == 0.0
    la, ph = B.amplitude(P, bits, 4)
    assert abs(la) < 1e-12


def test_amplitude_matches_statevector():
    """O6 in the exact regime: ln|<x|psi>| and its phase equal the dense amplitude."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 3, seed=4, xi=3.0)
    psi = SV.statevector(st)
    P = B.Prepared(st, lat.rows)
    rng = np.random.default_rng(1)
    for _ in range(5):
        x = rng.integers(0, 2, lat.n)
        idx = int("".join(map(str, x)), 2)
        la, ph = B.amplitude(P, x, 32)
        a = psi[idx]
        assert abs(la - math.log(abs(a))) < 1e-10
        assert abs(np.exp(1j * ph) - a / abs(a)) < 1e-10


def test_row_order_invariance_exact_regime():
    """in the exact regime reversing the rows leaves q(x) unchanged per x."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=6, xi=2.0)
    rows_rev = [list(reversed(r)) for r in reversed(lat.rows)]
    P1 = B.Prepared(st, lat.rows)
    P2 = B.Prepared(st, rows_rev)
    M1, _ = B.norm_envs(P1, 16)
    M2, _ = B.norm_envs(P2, 16)
    rng = np.random.default_rng(3)
    for _ in range(6):
        x = rng.integers(0, 2, lat.n)
        _, l1, _, _ = B.sample(P1, M1, 16, np.zeros(lat.n), forced=x)
        _, l2, _, _ = B.sample(P2, M2, 16, np.zeros(lat.n), forced=x)
        assert abs(l1 - l2) < 1e-10


def test_truncated_q_is_normalised_and_unbiased():
    """At finite R the sampled q is still a distribution (sum_x q = 1), so
    E_q[p/q] = sum_x p(x) = <psi|psi> holds exactly over the support."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 3, seed=9, xi=4.0)
    psi = SV.statevector(st)
    p = np.abs(psi) ** 2
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 2)
    qs = _all_q(P, M, 2, lat.n)
    assert abs(sum(qs.values()) - 1) < 1e-12
    est = sum(q * p[int("".join(map(str, x)), 2)] / q for x, q in qs.items() if q > 0)
    assert abs(est - p.sum()) < 1e-12 * p.sum()
    # and it is not the exact distribution (the truncation is real)
    pn = p / p.sum()
    assert max(abs(q - pn[int("".join(map(str, x)), 2)]) for x, q in qs.items()) > 1e-4


def test_row_validation():
    from oracle.rows import RowError, analyse
    lat = L.square(3, 3)
    analyse(lat.n, lat.edges, None, lat.rows)
    with pytest.raises(RowError):  # columns of a square lattice in a scrambled order
        analyse(lat.n, lat.edges, None, [[0, 4, 8], [1, 3, 5], [2, 6, 7]])
    with pytest.raises(RowError):  # not a permutation
        analyse(lat.n, lat.edges, None, [[0, 1, 2], [3, 4, 5], [6, 7, 7]])
    with pytest.raises(RowError):  # crossing inter-row edges
        analyse(lat.n, lat.edges, None, [[0, 1, 2], [5, 4, 3], [6, 7, 8]])


def test_kld_worked_example():
    from oracle import metrics
    rows = [l.split() for l in open(os.path.join(GOLDEN, "kld_arith.txt")) if l.strip() and not l.startswith("#")]
    q = [float(r[0]) for r in rows[:2]]
    p = [float(r[1]) for r in rows[:2]]
    want = float(rows[2][0])
    assert abs(metrics.kld(np.log(q), np.log(p)) - want) < 1e-15
    # identity observable -> 1 exactly
    assert abs(metrics.importance_expectation(np.log(q), np.log(p), [1, 1]) - 1) < 1e-15


# ---------------------------------------------------------------- NEXT-3: paper-literal order
def _all_q_literal(P, M, R, n):
    qs = {}
    for x in itertools.product([0, 1], repeat=n):
        bits, logq, cond, _ = B.sample_literal(P, M, R, np.zeros(n), forced=np.array(x))
        qs[x] = math.exp(logq)
    return qs


def test_literal_order_exact_regime_is_statevector():
    """the paper's own order (sample against the uncompressed m.psi_b, then
    fit) is exact when R is exact: q(x) = |<x|psi>|^2 / <psi|psi> for all 512 x of config 1
    and the drawn conditionals equal the statevector conditionals."""
    lat, st = G.config_state("cfg1")
    psi = SV.statevector(st)
    p = np.abs(psi) ** 2 / np.vdot(psi, psi).real
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 16)
    qs = _all_q_literal(P, M, 16, lat.n)
    for x, q in qs.items():
        assert abs(q - p[int("".join(map(str, x)), 2)]) < 1e-12
    u = S.uniforms(8, lat.n, 1001)
    for k in range(8):
        bits, logq, cond, fl = B.sample_literal(P, M, 16, u[k])
        ref = SV.conditionals(psi, lat.n, order_of(lat.rows), bits)
        assert np.allclose([cond[v] for v in order_of(lat.rows)], ref, rtol=1e-10)


def test_literal_order_truncated_is_normalised_and_differs():
    """At finite R the literal order's q is a distribution too (sum_x q = 1, so E_q[p/q] =
    <psi|psi>), and it differs from compress-then-sample (R3): the two
    orders coincide only in the exact regime."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 3, seed=9, xi=4.0)
    psi = SV.statevector(st)
    p = np.abs(psi) ** 2
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 2)
    ql = _all_q_literal(P, M, 2, lat.n)
    assert abs(sum(ql.values()) - 1) < 1e-12
    est = sum(q * p[int("".join(map(str, x)), 2)] / q for x, q in ql.items() if q > 0)
    assert abs(est - p.sum()) < 1e-12 * p.sum()
    qc = _all_q(P, M, 2, lat.n)
    assert max(abs(ql[x] - qc[x]) for x in ql) > 1e-6


def test_path_amplitude_is_exact_amplitude_in_exact_regime():
    """with fits that make no truncation, p(x) is the square of the MPS-MPS
    contraction m_{N_b-1 -> N_b} . X_{N_b} carried along the sampling path: ln|a| and arg a
    equal the brute-force statevector amplitude of every sampled bitstring (3x3, exact R)."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    psi = SV.statevector(st)
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 16)
    u = S.uniforms(10, lat.n, 6)
    for k in range(len(u)):
        bits, lq, _, _, (la, ph) = B.sample(P, M, 16, u[k], path_amplitude=True)
        a = psi[int("".join(map(str, bits)), 2)]
        assert abs(la - math.log(abs(a))) < 1e-9
        assert abs(np.exp(1j * (ph - np.angle(a))) - 1) < 1e-9
    # truncated (R = 2): the path amplitude is an approximation of <x|psi> (not exact)
    M2, _ = B.norm_envs(P, 2)
    errs = []
    for k in range(len(u)):
        bits, _, _, _, (la, _) = B.sample(P, M2, 2, u[k], path_amplitude=True)
        errs.append(abs(la - math.log(abs(psi[int("".join(map(str, bits)), 2)]))))
    assert max(errs) > 1e-6


# ---------------------------------------------------------------- NEXT-3: chip-row partition
def _chip_split(lat, st):
    rows = L.chip_rows(lat)
    return S.split_two_edge_vertices(st, rows, [c[0] for c in lat.coords])


def test_chip_row_partition_exact_regime_is_statevector():
    """The chip-row ("diagonal") partition of a rotated square patch, every interior
    vertex with two up and two down edges, through the vertex split (pure re-indexing,
    tninputs.synthetic.split_two_edge_vertices): exact regime -> the statevector conditionals
    and ln p of the qubits; the virtual vertices always draw 0 with conditional 1."""
    lat = L.rotated_patch(5, 5)
    st = S.vidal_like(lat, 2, seed=4, xi=2.0)
    st2, rows2, nq = _chip_split(lat, st)
    assert max(len([e for e in range(len(lat.edges)) if v in lat.edges[e]]) for v in range(lat.n)) == 4
    psi = SV.statevector(st)
    Z = np.vdot(psi, psi).real
    P = B.Prepared(st2, rows2)
    M, _ = B.norm_envs(P, 64)
    u = S.uniforms(6, st2["n"], 3)
    order = [v for r in rows2 for v in r if v < nq]
    for k in range(len(u)):
        bits, lq, cond, _ = B.sample(P, M, 64, u[k])
        assert (bits[nq:] == 0).all() and np.allclose(cond[nq:], 1.0)
        ref = SV.conditionals(psi, nq, order, bits[:nq])
        assert np.allclose([cond[v] for v in order], ref, atol=1e-10)
        assert abs(lq - math.log(abs(psi[int("".join(map(str, bits[:nq])), 2)]) ** 2 / Z)) < 1e-9


def test_chip_row_partition_truncated_is_normalised():
    """At finite R the chip-row sampler still defines a distribution: sum_x q(x) = 1 over all
    qubit bitstrings (virtual vertices forced to 0), and it differs from p (truncation is real)."""
    lat = L.rotated_patch(4, 4)
    st = S.vidal_like(lat, 3, seed=6, xi=3.0)
    st2, rows2, nq = _chip_split(lat, st)
    P = B.Prepared(st2, rows2)
    M, _ = B.norm_envs(P, 2)
    psi = SV.statevector(st)
    p = np.abs(psi) ** 2
    p /= p.sum()
    tot, diff = 0.0, 0.0
    for x in itertools.product([0, 1], repeat=nq):
        forced = np.zeros(st2["n"], dtype=np.uint8)
        forced[:nq] = x
        _, lq, _, _ = B.sample(P, M, 2, np.zeros(st2["n"]), forced=forced)
        q = math.exp(lq)
        tot += q
        diff = max(diff, abs(q - p[int("".join(map(str, x)), 2)]))
    assert abs(tot - 1) < 1e-10
    assert diff > 1e-6
