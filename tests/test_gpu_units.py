"""GPU unit tests of the building blocks (contraction engine, orthonormal bases) against a
plain numpy reference of the same operation (test-only debug entry points)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_11424_b200 import _lib  # noqa: E402

LIB = _lib.lib()
LIB.tn_debug_last_error.restype = C.c_char_p


def rand(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)


def dcontract(A, la, B, lb, lout, nb=1, perA=False, perB=False, cA=False, cB=False, gemm=0):
    shA = A.shape[1:] if perA else A.shape
    shB = B.shape[1:] if perB else B.shape
    A = np.ascontiguousarray(A, dtype=np.complex64)
    B = np.ascontiguousarray(B, dtype=np.complex64)
    ref = np.einsum(f"{'Q' if perA else ''}{la},{'Q' if perB else ''}{lb}->{'Q' if (perA or perB) else ''}{lout}",
                    A.conj() if cA else A, B.conj() if cB else B)
    out = np.zeros(ref.shape, dtype=np.complex64)
    sa = (C.c_int * len(shA))(*shA)
    sb = (C.c_int * len(shB))(*shB)
    rc = LIB.tn_debug_contract(la.encode(), len(shA), sa, A.ctypes.data_as(C.c_void_p), int(cA), int(perA),
                               lb.encode(), len(shB), sb, B.ctypes.data_as(C.c_void_p), int(cB), int(perB),
                               lout.encode(), nb, out.ctypes.data_as(C.c_void_p), C.c_int64(out.size), gemm)
    assert rc == 0, LIB.tn_debug_last_error()
    return out, ref


LIB.tn_debug_contract.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_char_p,
                                  C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_int,
                                  C.c_void_p, C.c_int64, C.c_int]
LIB.tn_debug_orth.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]


def close(a, b, tol=2e-5):
    return np.linalg.norm(a - b) <= tol * max(1e-30, np.linalg.norm(b))


@pytest.mark.parametrize("gemm", [1, 0, 2])
@pytest.mark.parametrize("case", [
    ("ab", (37, 29), "bc", (29, 41), "ac"),
    ("ab", (37, 29), "cb", (41, 29), "ca"),
    ("xmy", (5, 7, 3), "mun", (7, 4, 6), "xyun"),
    ("xyun", (5, 3, 4, 6), "upyr", (4, 9, 3, 2), "xnpr"),
    ("xnpr", (5, 6, 9, 2), "znr", (8, 6, 2), "xpz"),
    ("asZeD", (3, 2, 4, 5, 6), "AsDZ", (7, 2, 6, 4), "saeA"),
    ("xeab", (3, 4, 2, 2), "edDf", (4, 3, 3, 5), "xabdDf"),
])
def test_contract_shared(case, gemm):
    rng = np.random.default_rng(0)
    la, sa, lb, sb, lo = case
    out, ref = dcontract(rand(rng, sa), la, rand(rng, sb), lb, lo, gemm=gemm)
    assert close(out, ref)


@pytest.mark.parametrize("gemm", [1, 0, 2])
def test_contract_batched_and_conj(gemm):
    rng = np.random.default_rng(1)
    nb = 5
    A = rand(rng, (nb, 6, 7, 3))
    B = rand(rng, (7, 3, 4))
    out, ref = dcontract(A, "xmy", B, "myn", "xn", nb=nb, perA=True, gemm=gemm)
    assert close(out, ref)
    out, ref = dcontract(B, "myn", A, "xmy", "nx", nb=nb, perB=True, cA=True, gemm=gemm)
    assert close(out, ref)
    B2 = rand(rng, (nb, 7, 3, 4))
    out, ref = dcontract(A, "xmy", B2, "myn", "nx", nb=nb, perA=True, perB=True, cB=True, gemm=gemm)
    assert close(out, ref)
    # element-wise (batched) label + unit dims
    A3 = rand(rng, (nb, 2, 3, 1, 4))
    B3 = rand(rng, (nb, 5, 2, 1, 4))
    out, ref = dcontract(A3, "saez", B3, "Asuz", "saeA", nb=nb, perA=True, perB=True, cB=True, gemm=gemm)
    assert close(out, ref)


@pytest.mark.parametrize("gemm", [1, 2])
def test_contract_gather_views(gemm):
    """Operands whose M/K axes are interleaved (the tensor-core path gathers them)."""
    rng = np.random.default_rng(11)
    nb = 3
    A = rand(rng, (nb, 5, 6, 7))
    B = rand(rng, (5, 7, 8))
    out, ref = dcontract(A, "mxy", B, "myn", "xn", nb=nb, perA=True, gemm=gemm)
    assert close(out, ref)
    B2 = rand(rng, (nb, 5, 7, 8))
    out, ref = dcontract(A, "mxy", B2, "myn", "xn", nb=nb, perA=True, perB=True, cB=True, gemm=gemm)
    assert close(out, ref)
    Y2 = rand(rng, (nb, 3, 2, 4, 5, 6))
    N = rand(rng, (nb, 7, 2, 6, 4))
    out, ref = dcontract(Y2, "asZeD", N, "AsDZ", "saeA", nb=nb, perA=True, perB=True, cB=True, gemm=gemm)
    assert close(out, ref)
    X1 = rand(rng, (4, 3, 2, 5, 6, 7))
    Aop = rand(rng, (2, 9, 5, 3, 8))
    out, ref = dcontract(X1, "xabdDf", Aop, "sudar", "xbDfsur", gemm=gemm)
    assert close(out, ref)


@pytest.mark.parametrize("la,shape", [("kxj", (13, 70, 23)), ("kjx", (13, 23, 70)), ("xjk", (70, 23, 13))])
def test_contract_prep_ragged_tiles(la, shape):
    """Tensor-core operand preparation over several 32 x 128 gather tiles with ragged tails in
    both M (70) and K (13 * 23 = 299), for each contiguity of the A operand (M innermost, K
    innermost, split K axes), per-sample A and conjugated B."""
    rng = np.random.default_rng(21)
    nb = 2
    A = rand(rng, (nb,) + shape)
    B = rand(rng, (13, 23, 40))
    out, ref = dcontract(A, la, B, "kjn", "xn", nb=nb, perA=True, cB=True, gemm=2)
    assert close(out, ref)
    out, ref = dcontract(B, "kjn", A, la, "nx", nb=nb, perB=True, cA=True, gemm=2)
    assert close(out, ref)


def test_contract_tiny_rows_tensor_core():
    """Rows/columns of magnitude ~1e-40 (FP32 subnormal) next to O(1) ones: the FP16x3 path's
    power-of-two scaling must stay finite (a scale of 2^139 once overflowed to inf -> NaN)."""
    rng = np.random.default_rng(9)
    A = rand(rng, (256, 512))
    B = rand(rng, (512, 256))
    A[3] *= 1e-40
    A[7] = 0
    B[:, 5] *= 1e-40
    out, ref = dcontract(A, "mk", B, "kn", "mn", gemm=2)
    assert np.isfinite(out).all()
    assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()


def test_contract_large_k():
    rng = np.random.default_rng(2)
    out, ref = dcontract(rand(rng, (130, 1000)), "ak", rand(rng, (1000, 70)), "kb", "ab")
    assert close(out, ref, 1e-5)


def _orth(X, transpose=False):
    nb = X.shape[0]
    if transpose:
        n, m = X.shape[1], X.shape[2]
    else:
        m, n = X.shape[1], X.shape[2]
    X = np.ascontiguousarray(X, dtype=np.complex64)
    Q = np.zeros_like(X)
    Cm = np.zeros((nb, n, n), dtype=np.complex64)
    rc = LIB.tn_debug_orth(m, n, nb, X.ctypes.data_as(C.c_void_p), Q.ctypes.data_as(C.c_void_p),
                           Cm.ctypes.data_as(C.c_void_p), int(transpose))
    assert rc == 0, LIB.tn_debug_last_error()
    return Q, Cm


@pytest.mark.parametrize("m,n", [(64, 16), (300, 128), (40, 40), (8192, 128)])
def test_orth_full_rank(m, n):
    rng = np.random.default_rng(3)
    X = rand(rng, (3, m, n)) * np.logspace(0, -4, n)[None, None, :]
    Q, Cm = _orth(X)
    for b in range(3):
        q = Q[b].astype(np.complex128)
        assert np.abs(q.conj().T @ q - np.eye(n)).max() < 1e-5
        # span: X = Q (Q^H X)
        x = X[b].astype(np.complex128)
        assert np.linalg.norm(x - q @ (q.conj().T @ x)) < 1e-5 * np.linalg.norm(x)
        assert np.linalg.norm(x - q @ Cm[b]) < 1e-5 * np.linalg.norm(x)


def test_orth_rank_deficient():
    rng = np.random.default_rng(4)
    m, n, r = 200, 32, 5
    X = (rand(rng, (2, m, r)) @ rand(rng, (2, r, n))).astype(np.complex64)
    X[1] = 0
    Q, _ = _orth(X)
    for b in range(2):
        q = Q[b].astype(np.complex128)
        assert np.abs(q.conj().T @ q - np.eye(n)).max() < 1e-5
        x = X[b].astype(np.complex128)
        assert np.linalg.norm(x - q @ (q.conj().T @ x)) <= 1e-5 * max(1e-30, np.linalg.norm(x))


@pytest.mark.parametrize("transpose", [False, True])
def test_orth_mixed_batch(transpose):
    """One launch over a batch mixing full-rank, exactly rank-deficient, numerically
    rank-deficient (FP32-level noise on a rank-3 matrix) and zero matrices: every basis is
    orthonormal, contains span(X), and C reproduces X."""
    rng = np.random.default_rng(6)
    m, n = 1024, 16
    X = rand(rng, (5, m, n)).astype(np.complex128)
    X[1] = rand(rng, (m, 3)) @ rand(rng, (3, n))
    X[2] = rand(rng, (m, 3)) @ rand(rng, (3, n))
    X[2] += 3e-6 * np.abs(X[2]).max() * rand(rng, (m, n))
    X[3] = 0
    X[4] *= 1e12
    if transpose:
        X = np.ascontiguousarray(np.swapaxes(X, 1, 2))
    Q, Cm = _orth(X.astype(np.complex64), transpose=transpose)
    for b in range(5):
        q = Q[b].astype(np.complex128)
        x = X[b].astype(np.complex64).astype(np.complex128)
        assert np.isfinite(q).all() and np.isfinite(Cm[b]).all(), b
        if transpose:
            q, x, c = q.T, x.T, Cm[b].conj()
        else:
            c = Cm[b]
        assert np.abs(q.conj().T @ q - np.eye(n)).max() < 1e-5, b
        nx = max(1e-30, np.linalg.norm(x))
        assert np.linalg.norm(x - q @ (q.conj().T @ x)) <= 1e-5 * nx, b
        assert np.linalg.norm(x - q @ c.astype(np.complex128)) <= 1e-5 * nx, b


def test_orth_rows():
    rng = np.random.default_rng(5)
    X = rand(rng, (2, 24, 300))  # rows orthonormalised (right_orth)
    Q, Cm = _orth(X, transpose=True)
    for b in range(2):
        q = Q[b].astype(np.complex128)
        assert np.abs(q @ q.conj().T - np.eye(24)).max() < 1e-5
        x = X[b].astype(np.complex128)
        # X = C^H Q
        assert np.linalg.norm(x - Cm[b].conj().T @ q) < 1e-5 * np.linalg.norm(x)


LIB.tn_debug_fit.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_int64,
                             C.c_void_p, C.c_void_p, C.c_int]


def gpu_fit(strip, R, tag=1, b1=1, nh=2, gemm=0):
    from oracle import bmps as B
    W = strip.W
    dbl = strip.kind == "double"
    keep = []
    tshape = np.zeros(4 * W, dtype=np.int32)
    tptr = (C.c_void_p * W)()
    tb = np.zeros(W, dtype=np.int32)
    mshape = np.zeros(5 * W, dtype=np.int32)
    mptr = (C.c_void_p * W)()
    for j in range(W):
        t = np.ascontiguousarray(strip.tops[j], dtype=np.complex64)
        keep.append(t)
        tshape[4 * j: 4 * j + t.ndim] = t.shape
        tptr[j] = t.ctypes.data
        tb[j] = t.shape[0]
        m = np.ascontiguousarray(strip.mats[j], dtype=np.complex64)
        keep.append(m)
        mshape[5 * j: 5 * j + m.ndim] = m.shape
        mptr[j] = m.ctypes.data
    outc = np.asarray(strip.out, dtype=np.int32)
    cap = 1 << 22
    out = np.zeros(cap, dtype=np.complex64)
    shapes = np.zeros(4 * W, dtype=np.int32)
    logn = np.zeros(1)
    K = LIB.tn_debug_fit(int(dbl), W, tshape.ctypes.data, tptr, tb.ctypes.data, mshape.ctypes.data, mptr,
                         outc.ctypes.data, R, tag, b1, nh, B.DEFAULT_SEED, out.ctypes.data, cap,
                         shapes.ctypes.data, logn.ctypes.data, gemm)
    assert K >= 0, LIB.tn_debug_last_error()
    sites, off = [], 0
    for k in range(K):
        sh = [int(x) for x in shapes[4 * k: 4 * k + 4] if x]
        size = int(np.prod(sh))
        sites.append(out[off: off + size].reshape(sh).astype(np.complex128))
        off += size
    return sites, float(logn[0])


def _dense(sites):
    v = np.ones((1, 1))
    for s in sites:
        s = s.reshape(s.shape[0], -1, s.shape[-1])
        v = np.einsum("Pa,apb->Ppb", v, s).reshape(-1, s.shape[-1])
    return v.reshape(-1)


@pytest.mark.parametrize("R", [64, 3])
@pytest.mark.parametrize("gemm", [1, 0, 2])
def test_fit_single_matches_oracle(R, gemm):
    import math
    from oracle import bmps as B
    from tests.test_oracle import _random_strip
    rng = np.random.default_rng(7)
    strip = _random_strip(rng, W=5, chi=3, mu=3)
    so, lo = B.fit(strip, R=R, tag=1, b1=2)
    sg, lg = gpu_fit(strip, R, tag=1, b1=2, gemm=gemm)
    ref = _dense(so) * math.exp(lo)
    got = _dense(sg) * math.exp(lg)
    assert np.linalg.norm(got - ref) <= 1e-4 * np.linalg.norm(ref)


def test_fit_double_matches_oracle():
    import math
    from oracle import bmps as B
    from tninputs import lattices as L
    from tninputs import synthetic as S
    lat = L.square(3, 3)
    st = S.vidal_like(lat, 2, seed=3, xi=2.0)
    P = B.Prepared(st, lat.rows)
    for R in (16, 3):
        M, logs = B.norm_envs(P, R)
        # fit of row 1 (0-based) with M[1] from below, as in norm_envs
        row = P.rows[1]
        tops = B._tops_for_row(P, row, M[1], "down", "double")
        strip = B.Strip("double", tops, [P.A[v] for v in row], [P.has(v, "up") for v in row])
        so, lo = B.fit(strip, R, B.TAG_M, 2)
        sg, lg = gpu_fit(strip, R, tag=B.TAG_M, b1=2)
        ref = _dense(so) * math.exp(lo)
        got = _dense(sg) * math.exp(lg)
        assert np.linalg.norm(got - ref) <= 1e-4 * np.linalg.norm(ref), R


@pytest.mark.parametrize("n", [1, 2, 5])
def test_contract_thin_n(n):
    """Thin GEMMs (N <= 8, K >= 256) take the warp-per-row kernel: batched, conjugated,
    strided-K operands against numpy."""
    rng = np.random.default_rng(12)
    nb = 3
    A = rand(rng, (nb, 37, 300))
    B = rand(rng, (300, n))
    out, ref = dcontract(A, "mk", B, "kn", "mn", nb=nb, perA=True, cA=True, gemm=1)
    assert close(out, ref)
    A2 = rand(rng, (nb, 300, 41))  # K-major A (strided K in the GEMM view)
    out, ref = dcontract(A2, "km", B, "kn", "nm", nb=nb, perA=True, cB=True, gemm=1)
    assert close(out, ref)


# ---------------------------------------------------------------- metric-shape GEMMs
LIB.tn_debug_set_zc.argtypes = [C.c_int]


def _contract_only(A, la, B, lb, lout, out_shape, nb, perA, perB, gemm=0):
    """GPU contraction without a full reference (large shapes)."""
    shA = A.shape[1:] if perA else A.shape
    shB = B.shape[1:] if perB else B.shape
    out = np.zeros(out_shape, dtype=np.complex64)
    sa = (C.c_int * len(shA))(*shA)
    sb = (C.c_int * len(shB))(*shB)
    rc = LIB.tn_debug_contract(la.encode(), len(shA), sa, A.ctypes.data_as(C.c_void_p), 0, int(perA),
                               lb.encode(), len(shB), sb, B.ctypes.data_as(C.c_void_p), 0, int(perB),
                               lout.encode(), nb, out.ctypes.data_as(C.c_void_p), C.c_int64(out.size), gemm)
    assert rc == 0, LIB.tn_debug_last_error()
    return out


def _rand32(rng, shape):
    a = np.empty(shape, dtype=np.complex64)
    a.real = rng.standard_normal(shape, dtype=np.float32)
    a.imag = rng.standard_normal(shape, dtype=np.float32)
    return a


def test_gemm_ladder_shape_elementwise():
    """The dominant ladder GEMM at the metric shape (Y2 = Y1 . M_j: per sample
    M = 2R^2 = 32768, K = N = chi R = 4096, two samples folded into M = 65536, shared B), on
    the tcgen05 FP16x3 path, element-wise against an FP64 reference on sampled rows of both
    samples: max |dC| <= 1e-5 max |C_ref| per row (FP32-class accuracy of R24; K = 8192 real
    reduction through the chunk promotion). Rows carry magnitudes over 6 decades and the two
    samples differ by 1e3 (per-row / per-sample scaling)."""
    rng = np.random.default_rng(41)
    nb, M, K, N = 2, 32768, 4096, 4096
    A = _rand32(rng, (nb, M, K))
    A *= (10.0 ** rng.uniform(-6, 0, (nb, M, 1))).astype(np.float32)
    A[1] *= np.float32(1e-3)
    B = (_rand32(rng, (K, N)) / np.float32(64.0)).astype(np.complex64)
    out = _contract_only(A, "mk", B, "kn", "mn", (nb, M, N), nb, True, False, gemm=2)
    rows = rng.choice(M, 48, replace=False)
    Bd = B.astype(np.complex128)
    for q in range(nb):
        ref = A[q, rows].astype(np.complex128) @ Bd
        err = np.abs(out[q, rows] - ref).max(axis=1) / np.abs(ref).max(axis=1)
        print("ladder shape max elementwise rel err", q, err.max()); assert err.max() <= 1e-5, (q, err.max())
    assert np.isfinite(out).all()


@pytest.mark.parametrize("shape", [(512, 1024, 256), (300, 700, 130), (100, 600, 70)])
def test_gemm_block_scaling_cancellation(shape):
    """Per-(row, 128-complex-K block) scales of A and per-(column, block) scales of B: each row
    of A is O(1) on the first K block and 1e-9 on the rest; B's first block rows are zero for
    the even columns. C[:, even] then only sees the small blocks (values ~1e-9 of A's row
    maximum). One scale per row (or per sample) would leave those entries an absolute error
    ~2^-24 of the row maximum, i.e. O(1) relative; the block scales keep every element within
    1e-5 of FP64 relative to sum_k |a_k b_k| (tcgen05 forced; ragged M, N, K)."""
    M, K, N = shape
    rng = np.random.default_rng(47)
    A = _rand32(rng, (M, K))
    A[:, 128:] *= np.float32(1e-9)
    B = _rand32(rng, (K, N))
    B[:128, 0::2] = 0
    out = _contract_only(A, "mk", B, "kn", "mn", (M, N), 1, False, False, gemm=2)
    Ad, Bd = A.astype(np.complex128), B.astype(np.complex128)
    ref = Ad @ Bd
    bound = np.abs(Ad) @ np.abs(Bd)
    err = (np.abs(out - ref) / bound).max()
    print("block-scaling cancellation: max |dC| / sum|a||b|", err)
    assert err <= 1e-5, err


@pytest.mark.parametrize("zc", [0, 2, 1])
def test_gemm_per_sample_b_chunked(zc):
    """Contraction with per-sample B over a batched label (the N = 128 ladder closure Rs =
    Y2 . conj(n): M = R^2, K = chi R = 4096, batched over s and the samples):
    A planes built in chunks of zc batch elements (tn_debug_set_zc forces zc < nbz) give
    bitwise the same result as one chunk, element-wise within 1e-5 of FP64."""
    rng = np.random.default_rng(43)
    nb, M, K, N = 3, 2048, 4096, 128
    A = _rand32(rng, (nb, 2, M, K))
    B = _rand32(rng, (nb, 2, K, N))
    B[2] *= np.float32(1e-4)
    LIB.tn_debug_set_zc(zc)
    try:
        out = _contract_only(A, "sMk", B, "skN", "sMN", (nb, 2, M, N), nb, True, True, gemm=2)
        LIB.tn_debug_set_zc(0)
        ref0 = _contract_only(A, "sMk", B, "skN", "sMN", (nb, 2, M, N), nb, True, True, gemm=2)
    finally:
        LIB.tn_debug_set_zc(0)
    assert np.array_equal(out, ref0)
    ref = np.matmul(A.astype(np.complex128), B.astype(np.complex128))
    err = np.abs(out - ref).max(axis=-1) / np.abs(ref).max(axis=-1)
    print("per-sample-B max elementwise rel err", zc, err.max()); assert err.max() <= 1e-5, err.max()


LIB.tn_debug_set_3m.argtypes = [C.c_int]


@pytest.mark.parametrize("case", [
    # (la, shapeA, lb, shapeB, lout, nb, perA, perB, cA, cB)
    ("ak", (300, 600), "kb", (600, 200), "ab", 1, False, False, False, False),       # ragged M, N, K
    ("ak", (257, 1040), "kb", (1040, 129), "ab", 1, False, False, True, False),      # conj A, ragged
    ("sMk", (2, 260, 530), "skN", (2, 530, 70), "sMN", 3, True, True, False, True),  # batched B, conj B
    ("mk", (1024, 2048), "kn", (2048, 256), "mn", 2, True, False, False, False),     # folded batch, 2 segments
    ("ak", (256, 4096), "kb", (4096, 64), "ab", 1, False, False, False, False),      # split-K (few tiles)
])
def test_gemm_3m_forced_vs_numpy(case):
    """The 3M (Gauss) tensor-core path (three real products T1 = Ar Br, T2 = Ai Bi,
    T3 = (Ar + Ai)(Br + Bi), staggered TMEM accumulation segments) forced on every pair-kernel
    GEMM (tn_debug_set_3m(2)): element-wise against an FP64 reference (max |dC| <= 1e-5
    max |C| per row) on ragged tiles, conjugated operands, per-sample B, folded batches,
    several promotion segments and split-K."""
    la, sa, lb, sb, lout, nb, perA, perB, cA, cB = case
    rng = np.random.default_rng(17)
    A = _rand32(rng, ((nb,) + sa) if perA else sa)
    B = _rand32(rng, ((nb,) + sb) if perB else sb)
    LIB.tn_debug_set_3m(2)
    try:
        out, ref = dcontract(A, la, B, lb, lout, nb=nb, perA=perA, perB=perB, cA=cA, cB=cB, gemm=2)
    finally:
        LIB.tn_debug_set_3m(-1)
    Ad = A.astype(np.complex128).conj() if cA else A.astype(np.complex128)
    Bd = B.astype(np.complex128).conj() if cB else B.astype(np.complex128)
    q = "Q" if (perA or perB) else ""
    ref = np.einsum(f"{'Q' if perA else ''}{la},{'Q' if perB else ''}{lb}->{q}{lout}", Ad, Bd)
    err = (np.abs(out - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).max()
    print("3m", la, sa, lb, sb, "max elementwise rel err", err)
    assert np.isfinite(out).all() and err <= 1e-5, err
