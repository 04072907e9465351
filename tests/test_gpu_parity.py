"""GPU <-> oracle parity through the C ABI (libtnsample.so on a B200).

Same seeded inputs on both sides (tninputs), the oracle in complex128 (oracle/), the CUDA
path in complex64 with FP32/TF32x3 products; tolerances of R16 (tests/parity.py).
"""
import math

import numpy as np
import pytest

from tests.parity import amp_close, compare_samples, oracle_samples
from tninputs import lattices as L
from tninputs import synthetic as S

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_11424_b200 import TNState  # noqa: E402
from oracle import bmps as B  # noqa: E402
from oracle import generator as G  # noqa: E402
from oracle import statevector as SV  # noqa: E402


def order_of(rows):
    return [v for r in rows for v in r]


def _run(st, rows, R, u, gemm=0):
    g = TNState(st)
    if gemm:
        g.set_option("gemm", gemm)
    bits, logq, cond, flags = g.sample(rows, R, u, want_cond=True)
    return g, bits, logq, cond, flags


@pytest.mark.parametrize("gemm", [1, 0])
def test_exact_regime_square_vs_statevector(gemm):
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    psi = SV.statevector(st)
    u = S.uniforms(64, lat.n, 5)
    g, bits, logq, cond, flags = _run(st, lat.rows, 16, u, gemm)
    order = order_of(lat.rows)
    for k in range(len(u)):
        ref = SV.conditionals(psi, lat.n, order, bits[k])
        got = [cond[k, v] for v in order]
        assert np.allclose(got, ref, rtol=1e-4, atol=1e-6), (k, got, ref)
        idx = int("".join(map(str, bits[k])), 2)
        lp = math.log(abs(psi[idx]) ** 2 / np.vdot(psi, psi).real)
        assert abs(logq[k] - lp) <= 1e-4 * max(1, abs(lp))
    assert abs(g.log_norm(16) - math.log(np.vdot(psi, psi).real)) < 1e-4


def test_config1_vs_oracle():
    lat, st = G.config_state("cfg1")
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 16)
    u = S.uniforms(1024, lat.n, 1001)
    g, bits, logq, cond, flags = _run(st, lat.rows, 16, u)
    n_ref = 128
    rb, rl, rc = oracle_samples(P, M, 16, u, n_ref)
    rep = compare_samples(order_of(lat.rows), u[:n_ref], bits[:n_ref], logq[:n_ref], cond[:n_ref], rb, rl, rc)
    assert rep["compared"] > 0
    # U(1): every GPU sample in the domain wall's sector
    assert (bits.sum(axis=1) == sum(L.domain_wall_bits(lat))).all()


def test_config1_truncated_vs_oracle():
    """Finite chi_env (R=4 < exact rank): q is defined by the fits."""
    lat, st = G.config_state("cfg1")
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 4)
    u = S.uniforms(64, lat.n, 1001)
    g, bits, logq, cond, flags = _run(st, lat.rows, 4, u)
    rb, rl, rc = oracle_samples(P, M, 4, u)
    compare_samples(order_of(lat.rows), u, bits, logq, cond, rb, rl, rc)


def test_amplitude_vs_oracle():
    lat, st = G.config_state("cfg1")
    P = B.Prepared(st, lat.rows)
    g = TNState(st)
    g.prepare(lat.rows, 16)
    rng = np.random.default_rng(2)
    x = rng.integers(0, 2, (16, lat.n)).astype(np.uint8)
    x[:8] = 0
    for k in range(8):  # magnetisation-sector bitstrings (non-zero amplitudes)
        ones = rng.choice(lat.n, sum(L.domain_wall_bits(lat)), replace=False)
        x[k, ones] = 1
    la, ph = g.amplitude(x, 8)
    M, logs = B.norm_envs(P, 16)
    half_lnZ = 0.5 * B.log_norm(P, M, logs)
    sector = sum(L.domain_wall_bits(lat))
    n_rel = 0
    for k in range(len(x)):
        lr, pr = B.amplitude(P, x[k], 8)
        forbidden = int(x[k].sum()) != sector  # U(1): <x|psi> = 0 exactly
        n_rel += not forbidden
        assert amp_close(la[k], ph[k], lr, pr, forbidden, half_lnZ), (k, la[k], lr, ph[k], pr)
    assert n_rel >= 8


@pytest.mark.parametrize("lat_name,chi,K,R", [("willow105", 4, 2, 8), ("square4x4", 4, 3, 16)])
def test_branch_superposition_full_topology(lat_name, chi, K, R):
    from tests.test_oracle import closed_form_conditionals
    lat = L.by_name(lat_name)
    st = S.branch_superposition(lat, chi, K, seed=2)
    u = S.uniforms(8, lat.n, 77)
    g, bits, logq, cond, flags = _run(st, lat.rows, R, u)
    order = order_of(lat.rows)
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k])
        got = [cond[k, v] for v in order]
        for a, b_ in zip(got, ref):
            assert abs(a - b_) <= 1e-4 * b_ + (1e-6 if b_ < 1e-2 else 0), (k, got, ref)


def test_branch_superposition_willow_full_chi():
    """Full metric-config tensor shapes (Willow-105, every bond chi = 32, dense tensors) in the
    exact regime: K = 4 branches -> boundary ranks <= 4 (single) / 16 (double) <= chi_env = 16,
    so q(x) and every conditional have the closed form of the branch sum (maths, not the
    oracle). Exercises the tcgen05 path at chi = 32 GEMM shapes."""
    from tests.test_oracle import closed_form_conditionals
    lat = L.willow105()
    st = S.branch_superposition(lat, 32, 4, seed=11)
    u = S.uniforms(4, lat.n, 12)
    g, bits, logq, cond, flags = _run(st, lat.rows, 16, u)
    order = order_of(lat.rows)
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k])
        for v, r in zip(order, ref):
            assert abs(cond[k, v] - r) <= 1e-4 * r + (1e-6 if r < 1e-2 else 0), (k, v, cond[k, v], r)
        assert abs(logq[k] - sum(math.log(r) for r in ref)) <= 1e-4 * max(1, abs(logq[k]))


def test_branch_superposition_metric_shapes_exact():
    """Exact regime at the METRIC shapes (chi = 32, chi_env = 128): K = 11 branches on three
    full-width Willow-105 rows (widths 3, 5, 7) give single-layer boundary ranks <= 11 and
    double-layer ranks <= 121 <= chi_env, so the method is exact while every
    fit runs at D = 128 with rank-deficient completion (R7), the ladder GEMMs have the
    metric shapes (Y2 = Y1 M_j: M = 2R^2 per sample, K = N = chi R = 4096; the per-sample-B
    contractions batch-chunked) and K = 8192 real reductions use the 8-chunk promotion.
    Every conditional and ln q is compared with the closed form of the branch sum
    (maths, not the oracle), element-wise at R16."""
    from tests.test_oracle import closed_form_conditionals
    lat = L.row_strip(L.willow105(), 1, 4)
    st = S.branch_superposition(lat, 32, 11, seed=23)
    u = S.uniforms(3, lat.n, 29)
    g, bits, logq, cond, flags = _run(st, lat.rows, 128, u)
    order = order_of(lat.rows)
    assert (flags == 0).all()
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k])
        for v, r in zip(order, ref):
            assert abs(cond[k, v] - r) <= 1e-4 * r + (1e-6 if r < 1e-2 else 0), (k, v, cond[k, v], r)
        assert abs(logq[k] - sum(math.log(r) for r in ref)) <= 1e-4 * max(1, abs(logq[k]))


def test_branch_superposition_env256_plane_blocks_exact():
    """chi_env = 256 on three full-width Willow rows (chi = 32, K = 11 branches: exact, as in
    the metric-shape test): the ladder GEMMs' plane outputs then carry two scale blocks per inner
    K digit (the digit of 256 split into block x 128 rows of a CTA tile); every conditional and
    ln q against the closed form, and the plane path must have run."""
    import ctypes
    from paper_2507_11424_b200 import _lib
    from tests.test_oracle import closed_form_conditionals
    lat = L.row_strip(L.willow105(), 1, 4)
    st = S.branch_superposition(lat, 32, 11, seed=23)
    u = S.uniforms(2, lat.n, 41)
    _lib.lib().tn_debug_plane_gemms.restype = ctypes.c_int64
    _lib.lib().tn_debug_plane_gemms(1)
    g, bits, logq, cond, flags = _run(st, lat.rows, 256, u)
    assert _lib.lib().tn_debug_plane_gemms(1) > 0
    order = order_of(lat.rows)
    assert (flags == 0).all()
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k])
        for v, r in zip(order, ref):
            assert abs(cond[k, v] - r) <= 1e-4 * r + (1e-6 if r < 1e-2 else 0), (k, v, cond[k, v], r)
        assert abs(logq[k] - sum(math.log(r) for r in ref)) <= 1e-4 * max(1, abs(logq[k]))


def test_metric_shapes_batch_composition_bitwise():
    """The metric-shape ladder runs through the plane-output GEMMs (the ladder GEMMs write their
    closures' FP16 A planes and block scales from the epilogue; G1 -> G2 -> Lx chained, the
    samples on the GEMM batch index or folded into M): one batch of 4, batches of 1 and 3, and
    the same samples in another order give bitwise the same bits, ln q and conditionals per
    sample (results depend only on a sample's own uniforms). A state with
    every vertex at full bonds (Vidal-like) on three full-width Willow rows, chi = 32,
    chi_env = 128."""
    lat = L.row_strip(L.willow105(), 1, 4)
    st = S.vidal_like(lat, 32, seed=7, xi=8.0)
    u = S.uniforms(4, lat.n, 31)
    g = TNState(st)
    import ctypes
    from paper_2507_11424_b200 import _lib
    _lib.lib().tn_debug_plane_gemms.restype = ctypes.c_int64
    _lib.lib().tn_debug_plane_gemms(1)
    ref = g.sample(lat.rows, 128, u, want_cond=True)
    assert _lib.lib().tn_debug_plane_gemms(1) > 0  # the plane-output path ran
    for mb in (1, 3):
        g.set_option("max_batch", mb)
        got = g.sample(lat.rows, 128, u, want_cond=True)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b), mb
    g.set_option("max_batch", 0)
    perm = [2, 0, 3, 1]
    got = g.sample(lat.rows, 128, u[perm], want_cond=True)
    for a, b in zip(ref, got):
        assert np.array_equal(a[perm], b)
    assert np.isfinite(ref[1]).all()


def test_ghz_eagle():
    lat = L.eagle127()
    st = S.ghz(lat, chi=2)
    u = S.uniforms(16, lat.n, 3)
    g, bits, logq, cond, flags = _run(st, lat.rows, 4, u)
    for k in range(len(u)):
        assert len(set(bits[k].tolist())) == 1
        assert abs(logq[k] - math.log(0.5)) < 1e-5


def test_relabelled_rows_same_result():
    """General row orders through the C ABI: relabelling vertices changes nothing."""
    lat = L.square(3, 4)
    st = S.vidal_like(lat, 2, seed=1, xi=2.0)
    perm = list(np.random.default_rng(0).permutation(lat.n))
    st2, rows2 = S.relabel(st, lat.rows, perm)
    u = S.uniforms(16, lat.n, 9)
    u2 = np.zeros_like(u)
    for v in range(lat.n):
        u2[:, perm[v]] = u[:, v]
    _, b1, l1, c1, _ = _run(st, lat.rows, 16, u)
    _, b2, l2, c2, _ = _run(st2, rows2, 16, u2)
    for v in range(lat.n):
        assert (b1[:, v] == b2[:, perm[v]]).all()
    assert np.allclose(l1, l2, rtol=1e-5, atol=1e-6)


def test_batch_size_determinism():
    lat, st = G.config_state("cfg1")
    u = S.uniforms(40, lat.n, 4)
    g = TNState(st)
    b1, l1, _, _ = g.sample(lat.rows, 16, u)
    g.set_option("max_batch", 7)
    b2, l2, _, _ = g.sample(lat.rows, 16, u)
    assert (b1 == b2).all() and np.array_equal(l1, l2)


@pytest.mark.parametrize("gemm", [2, 0])
def test_batch_size_determinism_tensor_cores(gemm):
    """Results of a sample do not depend on which other samples share its batch (header:
    "results do not depend on batching or GPU count"): the tensor-core path (gemm = 2 forces
    it for every GEMM) scales produced operands per sample, so bits, ln q and every
    conditional are bitwise identical for max_batch in {1, 3, all}, on heterogeneous samples
    (config 2 quench state at finite chi_env, different branches per sample)."""
    lat, st = G.config_state("cfg2")
    u = S.uniforms(7, lat.n, 4)
    u[3] = 0.999  # an extreme sample in the middle of the batch
    g = TNState(st)
    g.set_option("gemm", gemm)
    ref = g.sample(lat.rows, 16, u, want_cond=True)
    for mb in (1, 3):
        g.set_option("max_batch", mb)
        got = g.sample(lat.rows, 16, u, want_cond=True)
        assert (got[0] == ref[0]).all(), mb
        assert np.array_equal(got[1], ref[1]), mb
        assert np.array_equal(got[2], ref[2]), mb
    # a sample alone equals the same sample inside a batch
    g.set_option("max_batch", 0)
    one = g.sample(lat.rows, 16, u[5:6], want_cond=True)
    assert (one[0][0] == ref[0][5]).all() and one[1][0] == ref[1][5]


def test_certify_matches_oracle_metrics():
    """tn_certify (NEXT-1): ln p from the GPU amplitude path equals the statevector;
    the weight statistics equal the oracle's metrics on the same (ln q, ln p)."""
    from oracle import metrics
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    psi = SV.statevector(st)
    u = S.uniforms(64, lat.n, 7)
    g, bits, logq, cond, flags = _run(st, lat.rows, 2, u)  # chi_env = 2 < exact: q != p
    lz = math.log(np.vdot(psi, psi).real)
    lp, stt = g.certify(bits, logq, 16, log_z=lz)
    for k in range(len(u)):
        idx = int("".join(map(str, bits[k])), 2)
        assert abs(lp[k] - math.log(abs(psi[idx]) ** 2)) < 1e-4 * max(1.0, abs(lp[k]))
    est, se = metrics.norm_estimate(logq, lp)
    assert abs(stt["log_norm_estimate"] - math.log(est)) < 1e-9
    assert abs(stt["norm_rel_stderr"] - se / est) < 1e-9
    assert abs(stt["kld"] - metrics.kld(logq, lp - lz)) < 1e-9
    r = np.exp(lp - logq)
    assert abs(stt["ess"] - r.sum() ** 2 / (r ** 2).sum()) < 1e-6 * len(r)
    assert stt["n_used"] == len(u) and stt["n_excluded"] == 0
    # unbiasedness: the estimate is within a few standard errors of <psi|psi>
    assert abs(math.exp(stt["log_norm_estimate"] - lz) - 1) < 5 * stt["norm_rel_stderr"] + 1e-6


def test_config2_vs_oracle():
    """BASELINE config 2 (6x6 square, domain-wall Heisenberg quench, 5 layers, chi = 8,
    chi_env = 32) at finite chi_env: per-sample conditionals, ln q and bits against the oracle
    (R16) on the same seeded state and uniforms; U(1) pass rate reported."""
    lat, st = G.config_state("cfg2")
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 32)
    u = S.uniforms(256, lat.n, 1002)
    g, bits, logq, cond, flags = _run(st, lat.rows, 32, u)
    rb, rl, rc = oracle_samples(P, M, 32, u, 8)
    rep = compare_samples(order_of(lat.rows), u[:8], bits[:8], logq[:8], cond[:8], rb, rl, rc)
    assert rep["compared"] > 0
    assert np.isfinite(logq).all() and (flags & 4 == 0).all()
    # truncation keeps the magnetisation sector for most samples (> 96 % at R = 3)
    ok = (bits.sum(axis=1) == sum(L.domain_wall_bits(lat))).mean()
    assert ok > 0.9, ok


def _run_literal(st, rows, R, u):
    g = TNState(st)
    g.set_option("order", 1)
    bits, logq, cond, flags = g.sample(rows, R, u, want_cond=True)
    return g, bits, logq, cond, flags


def test_literal_order_exact_regime_vs_statevector():
    """NEXT-3: the paper's own order on the GPU, exact regime -> the
    statevector conditionals and ln q."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    psi = SV.statevector(st)
    u = S.uniforms(32, lat.n, 5)
    g, bits, logq, cond, flags = _run_literal(st, lat.rows, 16, u)
    order = order_of(lat.rows)
    for k in range(len(u)):
        ref = SV.conditionals(psi, lat.n, order, bits[k])
        assert np.allclose([cond[k, v] for v in order], ref, rtol=1e-4, atol=1e-6), k
        idx = int("".join(map(str, bits[k])), 2)
        lp = math.log(abs(psi[idx]) ** 2 / np.vdot(psi, psi).real)
        assert abs(logq[k] - lp) <= 1e-4 * max(1, abs(lp))


@pytest.mark.parametrize("R", [4, 2])
def test_literal_order_truncated_vs_oracle(R):
    """NEXT-3 at finite chi_env (config 1 state): GPU vs oracle.sample_literal (R16)."""
    lat, st = G.config_state("cfg1")
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, R)
    u = S.uniforms(32, lat.n, 1001)
    g, bits, logq, cond, flags = _run_literal(st, lat.rows, R, u)
    rb = np.zeros((len(u), lat.n), np.uint8)
    rl = np.zeros(len(u))
    rc = np.zeros((len(u), lat.n))
    for k in range(len(u)):
        rb[k], rl[k], rc[k], _ = B.sample_literal(P, M, R, u[k])
    rep = compare_samples(order_of(lat.rows), u, bits, logq, cond, rb, rl, rc)
    assert rep["compared"] > 0


def test_literal_order_willow_topology():
    """NEXT-3 on the full Willow-105 topology (chi = 2, chi_env = 4) against the oracle."""
    lat = L.willow105()
    st = S.vidal_like(lat, 2, seed=21, xi=2.0)
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 4)
    u = S.uniforms(4, lat.n, 31)
    g, bits, logq, cond, flags = _run_literal(st, lat.rows, 4, u)
    rb = np.zeros((len(u), lat.n), np.uint8)
    rl = np.zeros(len(u))
    rc = np.zeros((len(u), lat.n))
    for k in range(len(u)):
        rb[k], rl[k], rc[k], _ = B.sample_literal(P, M, 4, u[k])
    compare_samples(order_of(lat.rows), u, bits, logq, cond, rb, rl, rc)


@pytest.mark.parametrize("shape", ["one_row", "one_column", "single_vertex"])
@pytest.mark.parametrize("order", [0, 1])
def test_degenerate_partitions_vs_statevector(shape, order):
    """Degenerate line partitions (SURVEY 8(c) edge cases): a chain as one row (no norm
    environments, no boundary MPS), a chain as one vertex per row (width-1 rows), a single
    qubit -- exact regime, both within-row orders, against the statevector."""
    from tninputs.lattices import Lattice
    n = 1 if shape == "single_vertex" else 6
    lat = L.chain(n)
    if shape == "one_row":
        lat = Lattice("chain_row", n, lat.edges, lat.coords, [list(range(n))], lat.colours)
    st = S.vidal_like(lat, 2, seed=4, xi=2.0)
    psi = SV.statevector(st)
    u = S.uniforms(16, lat.n, 8)
    g = TNState(st)
    if order:
        g.set_option("order", 1)
    bits, logq, cond, flags = g.sample(lat.rows, 8, u, want_cond=True)
    order_v = order_of(lat.rows)
    for k in range(len(u)):
        ref = SV.conditionals(psi, lat.n, order_v, bits[k])
        assert np.allclose([cond[k, v] for v in order_v], ref, rtol=1e-4, atol=1e-6), (k, shape)
    la, ph = g.amplitude(bits[:4], 8)
    for k in range(4):
        idx = int("".join(map(str, bits[k])), 2)
        assert abs(la[k] - math.log(abs(psi[idx]))) < 1e-4


# ------------------------------------------------------------------ oracle goldens (P1, w16)
GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


def _golden(name):
    import os
    path = os.path.join(GOLDEN, f"{name}_oracle.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (scripts/make_golden.py {name})")
    return np.load(path)


def test_p1_willow_quench_vs_oracle_golden():
    """P1 (SURVEY 8(d) parity aux): Willow-105, L = 15 domain-wall Heisenberg quench at chi = 8
    (the oracle generator's state rounded to complex64, tests/golden/p1_state.npz), chi_env = 32,
    64 samples: every conditional, ln q and bit against the CPU oracle's values
    (tests/golden/p1_oracle.npz, written by scripts/make_golden.py p1 -- oracle/ only), at R16."""
    import os
    ref = _golden("p1")
    st = S.load_state(os.path.join(GOLDEN, "p1_state.npz"))
    st["tensors"] = [np.asarray(t, dtype=np.complex128) for t in st["tensors"]]
    lat = L.willow105()
    R = int(ref["chi_env"])
    u = S.uniforms(len(ref["logq"]), lat.n, int(ref["uniform_seed"]))
    g, bits, logq, cond, flags = _run(st, lat.rows, R, u)
    rep = compare_samples(order_of(lat.rows), u, bits, logq, cond, ref["bits"], ref["logq"], ref["cond"])
    print("P1", rep)
    assert rep["compared"] >= 60 * lat.n
    assert abs(g.log_norm(R) - float(ref["log_norm"])) <= 1e-4 * abs(float(ref["log_norm"]))


def test_w16_willow_vs_oracle_golden():
    """Willow-105 at chi = 16, chi_env = 64 (Vidal-like state of the bench's recipe, seed 2507):
    the GPU against the CPU oracle's conditionals, ln q and bits (tests/golden/w16_oracle.npz,
    scripts/make_golden.py w16), at R16."""
    ref = _golden("w16")
    lat = L.willow105()
    st = S.vidal_like(lat, int(ref["chi"]), seed=2507)
    R = int(ref["chi_env"])
    u = S.uniforms(len(ref["logq"]), lat.n, int(ref["uniform_seed"]))
    g, bits, logq, cond, flags = _run(st, lat.rows, R, u)
    rep = compare_samples(order_of(lat.rows), u, bits, logq, cond, ref["bits"], ref["logq"], ref["cond"])
    print("w16", rep)
    assert rep["compared"] >= (len(u) - 1) * lat.n


# ------------------------------------------------------------------ configs 3 and 5 (topologies)
def test_cfg5_lucj_reduced_vs_oracle():
    """Config 5 topology (LUCJ-like 52-qubit two-register ladder, rows = rung pairs, PAPER.md:
    147-155) with the synthetic LUCJ circuit of the oracle generator (XX+YY brickwork, CP on the
    rungs, HF-like start) at reduced depth and bond (chi = 16, 4 + 4 layers) and chi_env = 16:
    every conditional, ln q and bit against the oracle (R16); particle number per register
    is conserved by every gate, so the samples lie in the HF sector."""
    lat, st = G.config_state("cfg5a", chi=16, layers=4)
    P = B.Prepared(st, lat.rows)
    R = 16
    M, _ = B.norm_envs(P, R)
    u = S.uniforms(48, lat.n, 1006)
    g, bits, logq, cond, flags = _run(st, lat.rows, R, u)
    rb, rl, rc = oracle_samples(P, M, R, u, 16)
    rep = compare_samples(order_of(lat.rows), u[:16], bits[:16], logq[:16], cond[:16], rb, rl, rc)
    assert rep["compared"] >= 15 * lat.n
    n_occ = G.LUCJ["cfg5a"][0]
    in_sector = ((bits[:, 0::2].sum(axis=1) == n_occ) & (bits[:, 1::2].sum(axis=1) == n_occ)).mean()
    print("cfg5 reduced", rep, "sector rate", in_sector)
    assert in_sector > 0.9


# ------------------------------------------------------------------ NEXT-1: path p, observables
def test_path_amplitude_vs_statevector_and_oracle():
    """tn_sample_path: exact regime -> ln|a| and arg a of every sample equal the
    statevector amplitude; truncated (config 1 state, chi_env = 4) -> equal to the oracle's
    path amplitude (oracle.bmps.sample(path_amplitude=True)) at R16."""
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    psi = SV.statevector(st)
    u = S.uniforms(32, lat.n, 6)
    g = TNState(st)
    bits, logq, la, ph = g.sample_path(lat.rows, 16, u)
    for k in range(len(u)):
        a = psi[int("".join(map(str, bits[k])), 2)]
        assert abs(la[k] - math.log(abs(a))) <= 1e-4 * max(1, abs(la[k]))
        assert abs(np.exp(1j * (ph[k] - np.angle(a))) - 1) <= 1e-4
    lat, st = G.config_state("cfg1")
    P = B.Prepared(st, lat.rows)
    M, _ = B.norm_envs(P, 4)
    u = S.uniforms(16, lat.n, 1001)
    g = TNState(st)
    bits, logq, la, ph = g.sample_path(lat.rows, 4, u)
    for k in range(len(u)):
        rb, rl, _, _, (ra, rp) = B.sample(P, M, 4, u[k], path_amplitude=True)
        if not (rb == bits[k]).all():
            continue  # a boundary case: the draw diverged (counted by the conditional tests)
        assert abs(la[k] - ra) <= 1e-4 * max(1, abs(ra)), (k, la[k], ra)
        assert abs(np.exp(1j * (ph[k] - rp)) - 1) <= 1e-4


def test_observables_vs_oracle_metrics():
    """tn_observables on GPU samples at finite chi_env with ln p from
    tn_certify: importance-sampled <Z_v> equals oracle.metrics.importance_expectation on the same
    (ln q, ln p, z_v); the sector pass rate equals the fraction of samples in the domain wall's
    magnetisation sector; with 512 samples the importance estimate of <Z_v> lies within 5
    standard errors of the statevector value."""
    from oracle import metrics
    from paper_2507_11424_b200 import observables
    lat, st = G.config_state("cfg1")
    psi = SV.statevector(st)
    u = S.uniforms(512, lat.n, 41)
    g = TNState(st)
    bits, logq, _, _ = g.sample(lat.rows, 4, u)
    lp, _ = g.certify(bits, logq, 16)
    target = sum(L.domain_wall_bits(lat))
    res = observables(bits, logq, lp, groups=[0] * lat.n, targets=[target])
    assert abs(res["pass_rate"] - (bits.sum(axis=1) == target).mean()) < 1e-12
    p = np.abs(psi) ** 2
    p /= p.sum()
    idx = np.arange(len(p))
    for v in range(lat.n):
        z = 1 - 2 * bits[:, v].astype(float)
        assert abs(res["z_weighted"][v] - metrics.importance_expectation(logq, lp, z)) < 1e-9
        assert abs(res["z_plain"][v] - z.mean()) < 1e-12
        zv = 1 - 2 * ((idx >> (lat.n - 1 - v)) & 1)
        exact = float((p * zv).sum())
        assert abs(res["z_weighted"][v] - exact) < 5 * 2 / math.sqrt(len(u)) + 1e-9


def test_cfg3_eagle_quench_vs_oracle_golden():
    """Config 3: IBM Eagle-127 heavy-hex domain-wall Heisenberg quench, L = 20,
    chi = 16 (the oracle generator's state rounded to complex64, tests/golden/cfg3_state.npz),
    chi_env = 64: conditionals, ln q and bits of 24 samples against the CPU oracle
    (tests/golden/cfg3_oracle.npz, scripts/make_golden.py cfg3), at R16; U(1) pass rate."""
    import os
    ref = _golden("cfg3")
    st = S.load_state(os.path.join(GOLDEN, "cfg3_state.npz"))
    st["tensors"] = [np.asarray(t, dtype=np.complex128) for t in st["tensors"]]
    lat = L.eagle127()
    R = int(ref["chi_env"])
    u = S.uniforms(len(ref["logq"]), lat.n, int(ref["uniform_seed"]))
    g, bits, logq, cond, flags = _run(st, lat.rows, R, u)
    rep = compare_samples(order_of(lat.rows), u, bits, logq, cond, ref["bits"], ref["logq"], ref["cond"])
    print("cfg3", rep, "U(1) pass", (bits.sum(axis=1) == sum(L.domain_wall_bits(lat))).mean())
    assert rep["compared"] >= (len(u) - 2) * lat.n


def test_cfg5_lucj_full_shapes_exact():
    """Config 5 at its full shapes (LUCJ-like 52-qubit two-register ladder, chi = 64,
    chi_env = 256, rows = rung pairs): K = 16 branches keep every single-layer boundary at rank
    <= 16 and every double-layer boundary at rank <= 256 = chi_env, so the method is exact
     and every conditional and ln q must equal the closed form of the branch sum."""
    from tests.test_oracle import closed_form_conditionals
    lat = L.by_name("lucj52")
    st = S.branch_superposition(lat, 64, 16, seed=31)
    u = S.uniforms(4, lat.n, 37)
    g, bits, logq, cond, flags = _run(st, lat.rows, 256, u)
    order = order_of(lat.rows)
    assert (flags == 0).all()
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k])
        for v, r in zip(order, ref):
            assert abs(cond[k, v] - r) <= 1e-4 * r + (1e-6 if r < 1e-2 else 0), (k, v, cond[k, v], r)
        assert abs(logq[k] - sum(math.log(r) for r in ref)) <= 1e-4 * max(1, abs(logq[k]))


# ------------------------------------------------------------------ NEXT-3: chip-row partition
def _chip(lat, st):
    return S.split_two_edge_vertices(st, L.chip_rows(lat), [c[0] for c in lat.coords])


def test_chip_row_partition_willow_exact_closed_form():
    """NEXT-3: the Willow-105 chip-row ("diagonal") partition -- 15 rows of 7
    qubits, two up and two down edges per interior qubit -- through the vertex split, on the GPU:
    a K = 3 branch superposition at chi = 4 (split bonds chi^2 = 16, chi_env = 32 >= every
    boundary rank) gives the closed-form conditionals of every qubit; virtual vertices draw 0.
    The branch factors phi_v^(c) have unit norm, so the three branches carry comparable weight:
    with unnormalised Gaussian factors (seed 5) branch 1 weighs 1.6e-5 of branch 0 over the
    lattice and less on partial products of rows, below the complex64 environments' resolution
    ("dynamic range"): the GPU then returns exactly the closed form of the
    two remaining branches (0.948771 vs 0.948645 at qubit 93)."""
    from tests.test_oracle import closed_form_conditionals
    lat = L.willow105()
    rng = np.random.default_rng(5)
    phis = rng.standard_normal((3, lat.n, 2)) + 1j * rng.standard_normal((3, lat.n, 2))
    phis /= np.linalg.norm(phis, axis=2, keepdims=True)
    st = S.branch_superposition(lat, 4, 3, seed=5, phis=phis)
    st2, rows2, nq = _chip(lat, st)
    u = S.uniforms(6, st2["n"], 19)
    g, bits, logq, cond, flags = _run(st2, rows2, 32, u)
    order = [v for r in rows2 for v in r if v < nq]
    assert (bits[:, nq:] == 0).all()
    for k in range(len(u)):
        ref = closed_form_conditionals(st["meta"]["phis"], order, bits[k, :nq])
        for v, r in zip(order, ref):
            assert abs(cond[k, v] - r) <= 1e-4 * r + (1e-6 if r < 1e-2 else 0), (k, v, cond[k, v], r)
        assert abs(logq[k] - sum(math.log(r) for r in ref)) <= 1e-4 * max(1, abs(logq[k]))


def test_chip_row_partition_vs_oracle_truncated():
    """NEXT-3 at finite chi_env: the chip-row partition of a Willow-105 quench state (chi = 2,
    3 layers) sampled at chi_env = 8 on the GPU against the oracle (R16), all conditionals."""
    lat = L.willow105()
    st = G.heisenberg_quench(lat, chi=2, layers=3)
    st2, rows2, nq = _chip(lat, st)
    P = B.Prepared(st2, rows2)
    M, _ = B.norm_envs(P, 8)
    u = S.uniforms(8, st2["n"], 23)
    g, bits, logq, cond, flags = _run(st2, rows2, 8, u)
    rb, rl, rc = oracle_samples(P, M, 8, u)
    rep = compare_samples([v for r in rows2 for v in r], u, bits, logq, cond, rb, rl, rc)
    print("chip rows", rep)
    assert rep["compared"] > 0
