"""ORACLE (test infrastructure only) -- generalised boundary-MPS sampling, complex128.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this
package; it shares no code with paper_2507_11424_b200/ (the CUDA path).

Plain, slow and step-by-step in the paper's order (App. "Sampling from
a Tensor Network State"), with the readings of SURVEY 8(c) listed in DESIGN.md:

* fit()             one-site variational MPS-MPO fit (Fig. 5c)  [O3]
* norm_envs()       M_{b+1->b} for b = N_b .. 2, once per state [O4]
* sample()          row-by-row, qubit-by-qubit conditionals, q(x)
                    as the product of the conditionals              [O5]
* amplitude()       <x|psi> by projected-row fits          [O6]
* log_norm()        <psi|psi> = <M_{2->1}, T_1> (R12)
* sample_literal()  the paper's own within-row order:
                    sample row b against the uncompressed m_{b-1} . psi_b, its conjugate
                    and M_{b+1->b} (a five-layer ladder), then fit m_b = Fit_R(m_{b-1} . X_b)

Notation: rows b = 0..N_b-1 (0-based here; the init hash uses the 1-based b of the
paper), columns j = 0..W_b-1 in row order, A_v[s, u, d, l, r] (SURVEY 8 notation).
Every contraction is pairwise (two operands per einsum, BLAS via optimize=True).
"""
from __future__ import annotations

import math

import numpy as np

from .rows import site_tensors

MASK64 = (1 << 64) - 1
DEFAULT_SEED = 0x2507114240
TAG_N, TAG_M, TAG_AMP, TAG_LIT = 1, 2, 3, 4


# ----------------------------------------------------------------------------- helpers
def pair(a, sa, b, sb, out):
    """One pairwise contraction (two operands only)."""
    return np.einsum(f"{sa},{sb}->{out}", a, b, optimize=True)


def splitmix64(x: int) -> int:
    """SplitMix64 finaliser of state x (the counter-based generator of O3)."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def hash_init(shape, seed: int, tag: int, b: int, k: int) -> np.ndarray:
    """Deterministic initial guess for output site k of the fit of row b (R4, O3):
    entry i (C order) = complex(h(2i), h(2i+1)), h = (SplitMix64(key) >> 40) * 2^-23 - 1,
    key = ((((seed*31 + tag)*1000003 + b)*1000003 + k)*4294967311 + 2i + c) mod 2^64."""
    base = ((((seed * 31 + tag) * 1000003 + b) * 1000003 + k) * 4294967311) & MASK64
    size = int(np.prod(shape))
    keys = np.uint64(base) + np.arange(2 * size, dtype=np.uint64)  # wraps mod 2^64
    h = splitmix64_np(keys)
    vals = (h >> np.uint64(40)).astype(np.float64) * 2.0 ** -23 - 1.0
    return (vals[0::2] + 1j * vals[1::2]).reshape(shape)


def splitmix64_np(x):
    """Vectorised SplitMix64 (uint64 arithmetic wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def left_orth(o):
    """Orthonormal basis of the column span of o reshaped (D_l * p) x D_r (one-site fit
    gauge move; R7: any orthonormal basis of the span)."""
    sh = o.shape
    q, _ = np.linalg.qr(o.reshape(-1, sh[-1]))
    return q.reshape(sh)


def right_orth(o):
    """Orthonormal basis of the row span of o reshaped D_l x (p * D_r), and the factor
    L with o = L . Q (returned for the gauge-preserving initial orthonormalisation)."""
    sh = o.shape
    x = o.reshape(sh[0], -1)
    q, r = np.linalg.qr(x.conj().T)
    return q.conj().T.reshape(sh), r.conj().T


# ----------------------------------------------------------------------------- strips
class Strip:
    """One row b of the network between an incoming boundary MPS ("top", one site per
    edge to the neighbouring row, identity where a column has no such edge) and the
    output MPS of the fit ("the MPO can be any tensor network which maps an
    MPS to another MPS").

    kind 'single': column j = top_j[m, u, n] x B_j[u, p, l, r]   (p open)
    kind 'double': column j = top_j[e, d, D, f] x A_j[s,u,d,l,r] x conj(A_j)[s,U,D,L,R]
                   (p = (u, U) open)
    out[j] says whether column j carries an output site; non-output columns have p of
    dimension 1 and are absorbed into the environments (R14 grouping).
    """

    def __init__(self, kind, tops, mats, out):
        self.kind = kind
        self.tops = tops
        self.mats = mats
        self.out = out
        self.W = len(mats)

    # bond dims ------------------------------------------------------------------------
    def top_bond_left(self, j):
        return self.tops[j].shape[0]

    def row_bond_left(self, j):
        return self.mats[j].shape[2] if self.kind == "single" else self.mats[j].shape[3]

    def cut_dim(self, j):
        """Dimension of the strip at the cut left of column j (top bond x row bond(s))."""
        r = self.row_bond_left(j)
        return self.top_bond_left(j) * (r if self.kind == "single" else r * r)

    def p_dim(self, j):
        if self.kind == "single":
            return self.mats[j].shape[1]
        u = self.mats[j].shape[1]
        return u * u

    def o_shape(self, j, dl, dr):
        if self.kind == "single":
            return (dl, self.p_dim(j), dr)
        u = self.mats[j].shape[1]
        return (dl, u, u, dr)

    def trivial_env(self):
        return np.ones((1, 1, 1) if self.kind == "single" else (1, 1, 1, 1), dtype=np.complex128)

    # transfer operations ---------------------------------------------------------------
    def _mid_single(self, L, j):
        X1 = pair(L, "xmy", self.tops[j], "mun", "xynu")
        return pair(X1, "xynu", self.mats[j], "upyr", "xnpr")

    def _mid_double(self, L, j, x0, x1):
        A = self.mats[j]
        X1 = pair(L[x0:x1], "xeab", self.tops[j], "edDf", "xabdDf")
        X2 = pair(X1, "xabdDf", A, "sudar", "xbDfsur")
        return pair(X2, "xbDfsur", A.conj(), "sUDbR", "xfurUR")

    def _chunks(self, L, j):
        """Slices of the output-bond index keeping double-layer intermediates bounded."""
        _, u, d, l, r = self.mats[j].shape
        f = self.tops[j].shape[3]
        per_x = max(l * l * d * d * f, 2 * l * d * f * u * r, f * u * u * r * r)
        per = max(1, int(4e7 // per_x))
        n = L.shape[0]
        return [(x, min(n, x + per)) for x in range(0, n, per)]

    def absorb_left(self, L, j, o):
        """L over columns < j  ->  L over columns <= j (o = output site of column j, or None)."""
        if self.kind == "single":
            X = self._mid_single(L, j)
            if o is None:
                return X[:, :, 0, :]
            return pair(X, "xnpr", o.conj(), "xpz", "znr")
        acc = None
        for x0, x1 in self._chunks(L, j):
            X = self._mid_double(L, j, x0, x1)
            if o is None:
                part = X[:, :, 0, :, 0, :]
            else:
                part = pair(X, "xfurUR", o[x0:x1].conj(), "xuUz", "zfrR")
            if o is None:
                acc = part if acc is None else np.concatenate([acc, part], axis=0)
            else:
                acc = part if acc is None else acc + part
        return acc

    def derivative(self, L, j, F):
        """o_j = d<o|T>/d conj(o_j) = L . (column j) . F."""
        if self.kind == "single":
            X = self._mid_single(L, j)
            return pair(X, "xnpr", F, "znr", "xpz")
        parts = []
        for x0, x1 in self._chunks(L, j):
            X = self._mid_double(L, j, x0, x1)
            parts.append(pair(X, "xfurUR", F, "zfrR", "xuUz"))
        return np.concatenate(parts, axis=0)

    def absorb_right(self, F, j, o, dl):
        """F over columns > j  ->  F over columns >= j."""
        top = self.tops[j]
        if self.kind == "single":
            B = self.mats[j]
            if o is None:
                Y1 = np.transpose(F, (1, 2, 0))[:, :, :, None]  # n r (x = z) p=1
            else:
                Y1 = pair(F, "znr", o.conj(), "xpz", "nrxp")
            Y2 = pair(Y1, "nrxp", B, "upyr", "nxuy")
            return pair(Y2, "nxuy", top, "mun", "xmy")
        A = self.mats[j]
        if o is None:
            Y1 = np.transpose(F, (1, 2, 3, 0))[:, :, :, :, None, None]  # f r R x u U
        else:
            Y1 = pair(F, "zfrR", o.conj(), "xuUz", "frRxuU")
        Y2 = pair(Y1, "frRxuU", A, "sudar", "fRxUsda")
        Y3 = pair(Y2, "fRxUsda", A.conj(), "sUDbR", "fxdaDb")
        return pair(Y3, "fxdaDb", top, "edDf", "xeab")


def identity_top(kind, bond):
    if kind == "single":
        return np.eye(bond, dtype=np.complex128).reshape(bond, 1, bond)
    return np.eye(bond, dtype=np.complex128).reshape(bond, 1, 1, bond)


def bond_dims(strip: Strip, R: int):
    """Output bonds D_0..D_K (D_0 = D_K = 1) by R6: min(R, strip cut dimension between
    consecutive output columns), then clamped so that D_k <= D_{k-1} p_k and
    D_{k-1} <= p_k D_k (which also enforces the products of physical dimensions)."""
    cols = [j for j in range(strip.W) if strip.out[j]]
    K = len(cols)
    D = [1] * (K + 1)
    for k in range(1, K):
        cut = min(strip.cut_dim(c) for c in range(cols[k - 1] + 1, cols[k] + 1))
        D[k] = min(R, cut)
    p = [strip.p_dim(c) for c in cols]
    for k in range(1, K):
        D[k] = min(D[k], D[k - 1] * p[k - 1])
    for k in range(K - 1, 0, -1):
        D[k] = min(D[k], p[k] * D[k + 1])
    return D


def fit(strip: Strip, R: int, tag: int, b1: int, seed: int = DEFAULT_SEED, nh: int = 2):
    """Fit_R of O3: one-site variational fit of the strip contraction T by an MPS of bond
    <= R. Returns (sites, log_norm); sites are normalised so that the
    fitted state is exp(log_norm) * |o>, |o> of unit norm. With no output column the
    strip is contracted exactly to a scalar and ([], log|s|, phase) semantics apply via
    the returned complex scalar in place of the site list."""
    cols = [j for j in range(strip.W) if strip.out[j]]
    K = len(cols)
    if K == 0:
        L = strip.trivial_env()
        for j in range(strip.W):
            L = strip.absorb_left(L, j, None)
        return L.reshape(-1)[0], 0.0
    D = bond_dims(strip, R)
    o = [hash_init(strip.o_shape(c, D[k], D[k + 1]), seed, tag, b1, k) for k, c in enumerate(cols)]
    # right-orthonormalise as a true gauge transformation (O3)
    for k in range(K - 1, 0, -1):
        q, l = right_orth(o[k])
        o[k] = q
        o[k - 1] = np.tensordot(o[k - 1], l, axes=([o[k - 1].ndim - 1], [0]))

    def env_left(Lk, k):
        L = strip.absorb_left(Lk, cols[k], o[k])
        end = cols[k + 1] if k + 1 < K else strip.W
        for j in range(cols[k] + 1, end):
            L = strip.absorb_left(L, j, None)
        return L

    def env_right(Fk, k):
        F = strip.absorb_right(Fk, cols[k], o[k], D[k])
        start = cols[k - 1] if k >= 1 else -1
        for j in range(cols[k] - 1, start, -1):
            F = strip.absorb_right(F, j, None, D[k])
        return F

    Lk = [None] * K
    Fk = [None] * K
    L = strip.trivial_env()
    for j in range(0, cols[0]):
        L = strip.absorb_left(L, j, None)
    Lk[0] = L
    F = strip.trivial_env()
    for j in range(strip.W - 1, cols[K - 1], -1):
        F = strip.absorb_right(F, j, None, 1)
    Fk[K - 1] = F
    for k in range(K - 1, 0, -1):
        Fk[k - 1] = env_right(Fk[k], k)

    for h in range(nh):
        if h % 2 == 0:  # left -> right
            for k in range(K):
                if not (h > 0 and k == 0):
                    o[k] = strip.derivative(Lk[k], cols[k], Fk[k])
                if k < K - 1:
                    o[k] = left_orth(o[k])
                    Lk[k + 1] = env_left(Lk[k], k)
        else:  # right -> left
            for k in range(K - 1, -1, -1):
                if k != K - 1:
                    o[k] = strip.derivative(Lk[k], cols[k], Fk[k])
                if k > 0:
                    o[k], _ = right_orth(o[k])
                    Fk[k - 1] = env_right(Fk[k], k)
    centre = K - 1 if nh % 2 == 1 else 0
    nrm = np.linalg.norm(o[centre])
    if nrm > 0:
        o[centre] = o[centre] / nrm
    return o, (math.log(nrm) if nrm > 0 else -math.inf)


# ----------------------------------------------------------------------------- the method
class Prepared:
    """A_v in [s,u,d,l,r] layout plus row structure for one (state, row order)."""

    def __init__(self, state, rows):
        self.state = state
        self.rows = [list(r) for r in rows]
        self.A, self.info = site_tensors(state, rows)
        self.n = state["n"]

    def has(self, v, key):
        return self.info[v][key] >= 0


def _tops_for_row(P: Prepared, row, mps, key, kind):
    """Place the sites of an incoming MPS on the columns that have an edge `key` ('up' for
    MPS from above, 'down' for norm MPS from below); identity elsewhere."""
    tops, k = [], 0
    bond = 1
    for v in row:
        if mps is not None and P.has(v, key):
            t = mps[k]
            k += 1
            tops.append(t)
            bond = t.shape[-1]
        else:
            tops.append(identity_top(kind, bond))
    if mps is not None:
        assert k == len(mps)
    return tops


def norm_envs(P: Prepared, R: int, seed: int = DEFAULT_SEED, nh: int = 2):
    """O4 / PAPER.md:279: M_{N_b} trivial; M_{b->b-1} = Fit_R(M_{b+1->b} . T_b), b = N_b..2.
    Returns (M, logs): M[b] is the norm MPS incident on row b from below (sites on the
    down-edge vertices of row b, [e, d, D, f]); M[N_b - 1] = None."""
    nb = len(P.rows)
    M = [None] * nb
    logs = [0.0] * nb
    for b in range(nb - 1, 0, -1):
        row = P.rows[b]
        tops = _tops_for_row(P, row, M[b], "down", "double")
        mats = [P.A[v] for v in row]
        out = [P.has(v, "up") for v in row]
        strip = Strip("double", tops, mats, out)
        sites, lg = fit(strip, R, TAG_M, b + 1, seed, nh)
        if isinstance(sites, list):
            M[b - 1] = sites
        else:
            M[b - 1] = None
        logs[b - 1] = lg
    return M, logs


def log_norm(P: Prepared, M, logs):
    """ln <psi|psi> ~ ln <M_{2->1}, T_1> plus the fit log-norms (R12)."""
    row = P.rows[0]
    tops = _tops_for_row(P, row, M[0], "down", "double")
    strip = Strip("double", tops, [P.A[v] for v in row], [False] * len(row))
    s, _ = fit(strip, 1, TAG_M, 1)
    return math.log(abs(s)) + sum(logs)


def _n_strip(P: Prepared, b, m_prev):
    row = P.rows[b]
    tops = _tops_for_row(P, row, m_prev, "up", "single")
    mats = []
    for v in row:
        A = P.A[v]  # [s,u,d,l,r]
        B = np.transpose(A, (1, 0, 2, 3, 4)).reshape(A.shape[1], 2 * A.shape[2], A.shape[3], A.shape[4])
        mats.append(B)
    return Strip("single", tops, mats, [True] * len(row))


def _merge(P: Prepared, row, sites, norms=None):
    """a5 / R14: slice s = x_v (done by the caller), multiply every vertex without a
    down-edge into the nearest down-edge site to its right, else to its left; normalise
    (the norms divided out are appended to `norms` when given)."""
    downs = [j for j, v in enumerate(row) if P.has(v, "down")]
    if not downs:
        return None
    out = []
    prev = -1
    for k, j in enumerate(downs):
        t = sites[j]  # [a, d, z]
        for i in range(j - 1, prev, -1):
            mat = sites[i][:, 0, :]
            t = np.tensordot(mat, t, axes=([1], [0]))
        if k == len(downs) - 1:
            for i in range(j + 1, len(row)):
                mat = sites[i][:, 0, :]
                t = np.tensordot(t, mat, axes=([2], [0]))
        prev = j
        nrm = np.linalg.norm(t)
        if norms is not None:
            norms.append(nrm)
        out.append(t / nrm)
    return out


def _row_scalar(sites):
    """Product of the projected sites [a, 1, b] of a row without down edges: the scalar the
    boundary contraction ends in (m_{N_b - 1 -> N_b} . X_{N_b})."""
    t = sites[0][:, 0, :]
    for x in sites[1:]:
        t = t @ x[:, 0, :]
    return complex(t.reshape(-1)[0])


def sample(P: Prepared, M, R: int, u_row, seed: int = DEFAULT_SEED, nh: int = 2, forced=None, max_rows=None,
           first_row=0, m_in=None, path_amplitude=False):
    """O5 for one sample: returns (bits[N] uint8 by vertex id, ln q, cond[N], flags).
    With `forced` (bits by vertex id) the draw is replaced by the given bits, which
    evaluates q(x) of any x (used to enumerate the whole distribution in tests).
    first_row / m_in / max_rows run rows first_row .. max_rows-1 only, starting from the
    incoming boundary MPS m_in (bounded CPU timing of a part of a sample only).
    path_amplitude: also return (ln|a|, arg a) of the amplitude carried along the sampling
    path, a = prod_b ||Fit(m_{b-1} psi_b)|| * ||merge(n_b[x_b])|| * (final scalar), i.e. the
    MPS-MPS contraction m_{N_b-1 -> N_b} . X_{N_b} whose square is p(x) when the fits are
    (near) exact (the first of its two ways to obtain p).

    Row b: n_b = Fit_R(m_{b-1} . psi_b) with (s, d) open (R3 compress-then-sample); right
    ladder R^(s)_j = n_j[s] M_j conj(n_j[s]) R_{j+1}; left pass w_s = Re<L_j, R^(s)_j>,
    clamp (R9), x = 0 iff u < P0 (R10), ln q += ln P(x);
    L_{j+1} = L_j n_j[x] M_j conj(n_j[x]); m_b = merge(n_b[x_b])."""
    n = P.n
    bits = np.zeros(n, dtype=np.uint8)
    cond = np.zeros(n, dtype=np.float64)
    logq = 0.0
    flags = 0
    m_prev = m_in
    log_amp, phase = 0.0, 0.0
    for b, row in enumerate(P.rows):
        if b < first_row:
            continue
        if max_rows is not None and b >= max_rows:  # partial run (bounded CPU timing only)
            break
        strip = _n_strip(P, b, m_prev)
        nsites, n_lg = fit(strip, R, TAG_N, b + 1, seed, nh)
        log_amp += n_lg
        W = len(row)
        ns = []
        for j, v in enumerate(row):
            dd = P.A[v].shape[2]
            t = nsites[j]
            ns.append(t.reshape(t.shape[0], 2, dd, t.shape[2]))  # [a, s, d, z]
        Ms = _tops_for_row(P, row, M[b], "down", "double")
        # right pass
        Rr = [None] * (W + 1)
        Rs = [None] * W
        Rr[W] = np.ones((1, 1, 1), dtype=np.complex128)
        for j in range(W - 1, -1, -1):
            Y1 = pair(ns[j], "asdz", Rr[j + 1], "zfZ", "asdfZ")
            Y2 = pair(Y1, "asdfZ", Ms[j], "edDf", "asZeD")
            Rs[j] = [pair(Y2[:, s], "aZeD", ns[j][:, s].conj(), "ADZ", "aeA") for s in range(2)]
            tot = Rs[j][0] + Rs[j][1]
            scale = np.abs(tot).max()
            Rr[j] = tot / scale if scale > 0 else tot
        # left pass
        Lx = np.ones((1, 1, 1), dtype=np.complex128)
        for j, v in enumerate(row):
            w = [float(np.real(np.sum(Lx * Rs[j][s]))) for s in range(2)]
            if w[0] < 0 or w[1] < 0:
                flags |= 1
            w = [max(x, 0.0) for x in w]
            tot = w[0] + w[1]
            if tot > 0:
                p0 = w[0] / tot
            else:
                flags |= 2
                p0 = 0.5
            if forced is None:
                x = 0 if u_row[v] < p0 else 1
            else:
                x = int(forced[v])
            px = p0 if x == 0 else 1.0 - p0
            bits[v] = x
            cond[v] = px
            logq += math.log(px) if px > 0 else -math.inf
            G1 = pair(Lx, "aeA", ns[j][:, x], "adz", "eAdz")
            G2 = pair(G1, "eAdz", Ms[j], "edDf", "AzDf")
            Lx = pair(G2, "AzDf", ns[j][:, x].conj(), "ADZ", "zfZ")
            scale = np.abs(Lx).max()
            if scale > 0:
                Lx = Lx / scale
        proj = [ns[j][:, bits[v]] for j, v in enumerate(row)]
        norms = []
        m_prev = _merge(P, row, proj, norms)
        log_amp += sum(math.log(x) if x > 0 else -math.inf for x in norms)
        if m_prev is None:  # no down edges: the boundary contraction ends in a scalar
            sc = _row_scalar(proj)
            log_amp += math.log(abs(sc)) if sc != 0 else -math.inf
            phase = math.atan2(sc.imag, sc.real)
    if path_amplitude:
        return bits, logq, cond, flags, (log_amp, phase)
    return bits, logq, cond, flags


def amplitude(P: Prepared, bits, R: int, seed: int = DEFAULT_SEED, nh: int = 2):
    """O6: <x|psi> by fitting m_b = Fit_R(m_{b-1} . psi_b[x_b]) with the down legs open
    (PAPER.md:85, 114, 293). Returns (ln|amp|, phase)."""
    m_prev = None
    logs = 0.0
    for b, row in enumerate(P.rows):
        tops = _tops_for_row(P, row, m_prev, "up", "single")
        mats = [np.transpose(P.A[v][int(bits[v])], (0, 1, 2, 3)) for v in row]  # [u, d, l, r]
        out = [P.has(v, "down") for v in row]
        strip = Strip("single", tops, mats, out)
        res, lg = fit(strip, R, TAG_AMP, b + 1, seed, nh)
        if isinstance(res, list):
            m_prev = res
            logs += lg
        else:
            s = complex(res)
            if s == 0:
                return -math.inf, 0.0
            return logs + math.log(abs(s)), math.atan2(s.imag, s.real)
    raise RuntimeError("last row has down edges")


def sample_literal(P: Prepared, M, R: int, u_row, seed: int = DEFAULT_SEED, nh: int = 2, forced=None):
    """NEXT-3: the paper's literal order. Row b is sampled qubit by qubit
    from the one-site reduced density matrices of the five-layer ladder
    m_{b-1->b} . psi_b . conj(psi_b) . conj(m_{b-1->b}) . M_{b+1->b} (sampled qubits projected
    on both layers, later ones traced), then m_{b->b+1} = Fit_R(m_{b-1->b} . X_b) with
    X_b = x_b . psi_b and the down legs open (tag 4). Same draw rule, clamp and ln q as
    sample() (R9, R10). Exact when R_x, R_n are exact.
    Right env R_j[a, l, L, A, e]: m bond, ket / bra row bond, conj(m) bond, M bond."""
    n = P.n
    bits = np.zeros(n, dtype=np.uint8)
    cond = np.zeros(n, dtype=np.float64)
    logq = 0.0
    flags = 0
    m_prev = None
    for b, row in enumerate(P.rows):
        W = len(row)
        ms = _tops_for_row(P, row, m_prev, "up", "single")     # [a, u, b] (identity: u = 1)
        Ms = _tops_for_row(P, row, M[b], "down", "double")     # [e, d, D, f]
        As = [P.A[v] for v in row]                              # [s, u, d, l, r]

        def right_site(R_next, j, s=None):
            # R_next[b, r, R, B, f] -> R_j[(s,) a, l, L, A, e]
            T1 = pair(R_next, "brRBf", ms[j], "aub", "rRBfau")
            T2 = pair(T1, "rRBfau", As[j], "sudlr", "RBfasdl")
            T3 = pair(T2, "RBfasdl", Ms[j], "edDf", "RBasleD")
            T4 = pair(T3, "RBasleD", As[j].conj(), "sUDLR", "sBaleUL")
            T5 = pair(T4, "sBaleUL", ms[j].conj(), "AUB", "salLAe")
            return T5 if s is None else T5[s]

        Rs = [None] * W
        Rr = np.ones((1, 1, 1, 1, 1), dtype=np.complex128)
        for j in range(W - 1, -1, -1):
            Rs[j] = right_site(Rr, j)                           # [s, a, l, L, A, e]
            tot = Rs[j][0] + Rs[j][1]
            scale = np.abs(tot).max()
            Rr = tot / scale if scale > 0 else tot  # [a, l, L, A, e] = [b, r, R, B, f] of column j-1
        Lx = np.ones((1, 1, 1, 1, 1), dtype=np.complex128)      # [a, l, L, A, e]
        for j, v in enumerate(row):
            w = [float(np.real(np.sum(Lx * Rs[j][s]))) for s in range(2)]
            if w[0] < 0 or w[1] < 0:
                flags |= 1
            w = [max(x, 0.0) for x in w]
            tot = w[0] + w[1]
            if tot > 0:
                p0 = w[0] / tot
            else:
                flags |= 2
                p0 = 0.5
            x = (0 if u_row[v] < p0 else 1) if forced is None else int(forced[v])
            px = p0 if x == 0 else 1.0 - p0
            bits[v] = x
            cond[v] = px
            logq += math.log(px) if px > 0 else -math.inf
            # L_{j+1}[b, r, R, B, f] = L_j . m_j . A_j[x] . M_j . conj(A_j[x]) . conj(m_j)
            G1 = pair(Lx, "alLAe", ms[j], "aub", "lLAeub")
            G2 = pair(G1, "lLAeub", As[j][x], "udlr", "LAebdr")
            G3 = pair(G2, "LAebdr", Ms[j], "edDf", "LAbrDf")
            G4 = pair(G3, "LAbrDf", As[j][x].conj(), "UDLR", "AbrfUR")
            Lx = pair(G4, "AbrfUR", ms[j].conj(), "AUB", "brRBf")
            scale = np.abs(Lx).max()
            if scale > 0:
                Lx = Lx / scale
        if b + 1 < len(P.rows):
            mats = [P.A[v][int(bits[v])] for v in row]                       # [u, d, l, r]
            out = [P.has(v, "down") for v in row]
            res, _ = fit(Strip("single", ms, mats, out), R, TAG_LIT, b + 1, seed, nh)
            m_prev = res if isinstance(res, list) else None
    return bits, logq, cond, flags

