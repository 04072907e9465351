"""ORACLE (test infrastructure only) -- TNS construction by BP-gauged simple update (O7).

Builds the configs' states the way the paper does:
* belief propagation on the norm network (R20: identity-initialised,
  normalised messages, synchronous sweeps, tol 1e-10, cap 50);
* two-qubit gates applied "by gauging the region with the square root of the incoming
  message tensors, applying the gate, performing a singular value decomposition, and
  ungauging the region with the inverse square root", truncating to chi
   and recording eps_i = discarded sum sigma^2 / sum sigma^2 (Eq. 1);
  f = prod (1 - eps_i) (Eq. 2);
* BP re-run between layers of non-overlapping gates, i.e. before every
  colour group of a Trotter step;
* Heisenberg Trotter gates exp(-i H_ij dt), H_ij = J(XX+YY+ZZ) (R22).
"""
from __future__ import annotations

import numpy as np

from tninputs import lattices as L
from tninputs import synthetic as S


def heisenberg_gate(J: float, dt: float) -> np.ndarray:
    """exp(-i J dt (XX+YY+ZZ)) = e^{i theta}[cos 2theta I - i sin 2theta SWAP], theta = J dt
    (R22; since XX+YY+ZZ = 2 SWAP - I). Index = 2 x_u + x_v (u < v)."""
    th = J * dt
    swap = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)
    return np.exp(1j * th) * (np.cos(2 * th) * np.eye(4) - 1j * np.sin(2 * th) * swap)


def xxpyy_gate(theta: float) -> np.ndarray:
    """XX+YY(theta) = exp(-i theta/4 (XX+YY)) (R22)."""
    c, s = np.cos(theta / 2), np.sin(theta / 2)
    return np.array([[1, 0, 0, 0], [0, c, -1j * s, 0], [0, -1j * s, c, 0], [0, 0, 0, 1]], dtype=np.complex128)


def cphase_gate(phi: float) -> np.ndarray:
    return np.diag([1, 1, 1, np.exp(1j * phi)]).astype(np.complex128)


class TNS:
    def __init__(self, lat, bits):
        self.lat = lat
        self.n = lat.n
        self.edges = [tuple(e) for e in lat.edges]
        self.inc = S.incident_edges(lat.n, lat.edges)
        st = S.product_state(lat, bits)
        self.t = [x.copy() for x in st["tensors"]]
        self.dims = [1] * len(self.edges)
        self.msg = {}
        self.eps = []

    def leg(self, v, e):
        return 1 + self.inc[v].index(e)

    # ---------------------------------------------------------------- belief propagation
    def _update(self, v, e, msg):
        """mu_{v->w} on edge e: contract A_v, conj(A_v) and every incoming message except the
        one on e, then normalise."""
        t = self.t[v]
        tt = t
        for e2 in self.inc[v]:
            if e2 == e:
                continue
            u = self.edges[e2][0] if self.edges[e2][1] == v else self.edges[e2][1]
            m = msg[(u, e2)]  # [k, k']
            ax = self.leg(v, e2)
            tt = np.moveaxis(np.tensordot(tt, m, axes=([ax], [0])), -1, ax)
        ax = self.leg(v, e)
        others = [i for i in range(t.ndim) if i != ax]
        out = np.tensordot(tt, t.conj(), axes=(others, others))
        out = 0.5 * (out + out.conj().T)
        return out / np.linalg.norm(out)

    def bp(self, tol=1e-10, max_sweeps=50):
        msg = {}
        for e, (u, w) in enumerate(self.edges):
            d = self.dims[e]
            msg[(u, e)] = np.eye(d, dtype=np.complex128) / np.sqrt(d)
            msg[(w, e)] = np.eye(d, dtype=np.complex128) / np.sqrt(d)
        res = np.inf
        for _ in range(max_sweeps):
            new = {}
            for e, (u, w) in enumerate(self.edges):
                new[(u, e)] = self._update(u, e, msg)
                new[(w, e)] = self._update(w, e, msg)
            res = max(np.linalg.norm(new[k] - msg[k]) for k in msg)
            msg = new
            if res < tol:
                break
        self.msg = msg
        return res

    # ---------------------------------------------------------------- gauged simple update
    @staticmethod
    def _sqrt_pair(m, cut=1e-12):
        lam, V = np.linalg.eigh(0.5 * (m + m.conj().T))
        lam = np.clip(lam, 0, None)
        keep = lam > cut * lam.max()
        sq = (V * np.sqrt(lam)) @ V.conj().T
        inv = np.zeros_like(lam)
        inv[keep] = 1 / np.sqrt(lam[keep])
        isq = (V * inv) @ V.conj().T
        return sq, isq

    def apply2(self, e, G, chi, cutoff=1e-14):
        v, w = self.edges[e]  # v < w; gate index 2 x_v + x_w
        sides = {}
        for a in (v, w):
            t = self.t[a]
            inv = {}
            for e2 in self.inc[a]:
                if e2 == e:
                    continue
                o = self.edges[e2][0] if self.edges[e2][1] == a else self.edges[e2][1]
                sq, isq = self._sqrt_pair(self.msg[(o, e2)])
                ax = self.leg(a, e2)
                t = np.moveaxis(np.tensordot(t, sq, axes=([ax], [0])), -1, ax)
                inv[ax] = isq
            ax_e = self.leg(a, e)
            others = [i for i in range(1, t.ndim) if i != ax_e]
            tp = np.transpose(t, others + [0, ax_e])
            osh = tp.shape[: len(others)]
            mat = tp.reshape(int(np.prod(osh)) if others else 1, 2 * t.shape[ax_e])
            Q, Rr = np.linalg.qr(mat)
            sides[a] = (Q, Rr.reshape(-1, 2, t.shape[ax_e]), others, osh, inv, t.ndim)
        Qv, rv, ov, oshv, invv, ndv = sides[v]
        Qw, rw, ow, oshw, invw, ndw = sides[w]
        theta = np.einsum("asx,btx->astb", rv, rw)
        g = G.reshape(2, 2, 2, 2)
        theta = np.einsum("stuv,auvb->astb", g, theta)
        qa, qb = theta.shape[0], theta.shape[3]
        U, sig, Vh = np.linalg.svd(theta.reshape(qa * 2, 2 * qb), full_matrices=False)
        w2 = sig ** 2
        tot = w2.sum()
        keep = int(min(chi, max(1, np.count_nonzero(w2 / tot > cutoff))))
        self.eps.append(float(w2[keep:].sum() / tot))
        sig = sig[:keep]
        U = U[:, :keep] * np.sqrt(sig)
        Vh = np.sqrt(sig)[:, None] * Vh[:keep]
        rv_new = U.reshape(qa, 2, keep)
        rw_new = Vh.reshape(keep, 2, qb).transpose(2, 1, 0)  # [b, t, x]
        for a, Q, rn, others, osh, inv, nd in ((v, Qv, rv_new, ov, oshv, invv, ndv),
                                               (w, Qw, rw_new, ow, oshw, invw, ndw)):
            t = (Q @ rn.reshape(rn.shape[0], -1)).reshape(tuple(osh) + (2, keep))
            # back to (s, legs in edge-id order)
            ax_e = self.leg(a, e)
            perm_src = others + [0, ax_e]
            t = np.transpose(t, np.argsort(perm_src))
            for ax, isq in inv.items():
                t = np.moveaxis(np.tensordot(t, isq, axes=([ax], [0])), -1, ax)
            self.t[a] = t / np.linalg.norm(t)
        self.dims[e] = keep
        d = np.diag(sig.astype(np.complex128))
        d = d / np.linalg.norm(d)
        self.msg[(v, e)] = d
        self.msg[(w, e)] = d

    def state(self, chi, meta):
        f = float(np.prod([1 - x for x in self.eps]))
        m = dict(meta)
        m.update({"eps": np.asarray(self.eps), "fidelity": f})
        return S.make_state(self.lat, self.t, self.dims, chi, m)


def heisenberg_quench(lat, chi: int, layers: int, J: float = 1.0, dt: float = 0.1):
    """Domain-wall quench: |0> on one half, |1> on the other (R18),
    L first-order Trotter layers over the lattice's colour groups."""
    tns = TNS(lat, L.domain_wall_bits(lat))
    G = heisenberg_gate(J, dt)
    residuals = []
    for _ in range(layers):
        for group in lat.colours:
            residuals.append(tns.bp())
            for e in group:
                tns.apply2(e, G, chi)
    return tns.state(chi, {"kind": "heisenberg", "layers": layers, "J": J, "dt": dt,
                            "bp_residual_max": float(max(residuals) if residuals else 0.0)})


def lucj_circuit(lat, chi: int, n_occ: int, rot_layers: int, seed: int):
    """Synthetic LUCJ-like circuit on a two-register ladder (config 5, SURVEY 8(d), R22;
    PAPER.md:147-151: "particle number preserving rotations - most prominently
    controlled-phase gates and XX + YY rotations"; the real circuits are not public,
    PAPER.md:234). Initial state HF-like: the first n_occ qubits of each register |1>, the
    rest |0> (R18-style reconstruction). Circuit: rot_layers brickwork layers of XX+YY(theta)
    on both register chains (even bonds, then odd bonds; an orbital-rotation network), one
    CP(phi) layer on every rung (the Jastrow part: "one or two control-phase gates per
    sub-register connection"), rot_layers more brickwork layers;
    theta, phi ~ U[-pi, pi) from default_rng(seed). BP refresh before every layer of
    non-overlapping gates."""
    n_reg = lat.n // 2
    bits = [1 if (v // 2) < n_occ else 0 for v in range(lat.n)]
    tns = TNS(lat, bits)
    rng = np.random.default_rng(seed)
    chain = {}
    rungs = []
    for e, (u, v) in enumerate(lat.edges):
        if v - u == 2:
            chain[(u, v)] = e
        else:
            rungs.append(e)
    alpha = [chain[(2 * i, 2 * i + 2)] for i in range(n_reg - 1)]
    beta = [chain[(2 * i + 1, 2 * i + 3)] for i in range(n_reg - 1)]
    residuals = []

    def rot_layer():
        for parity in (0, 1):
            group = [e for i, e in enumerate(alpha) if i % 2 == parity] + \
                    [e for i, e in enumerate(beta) if i % 2 == parity]
            residuals.append(tns.bp())
            for e in group:
                tns.apply2(e, xxpyy_gate(rng.uniform(-np.pi, np.pi)), chi)

    for _ in range(rot_layers):
        rot_layer()
    residuals.append(tns.bp())
    for e in rungs:
        tns.apply2(e, cphase_gate(rng.uniform(-np.pi, np.pi)), chi)
    for _ in range(rot_layers):
        rot_layer()
    n_gates = 2 * rot_layers * (len(alpha) + len(beta))
    return tns.state(chi, {"kind": "lucj", "n_occ": n_occ, "rot_layers": rot_layers, "seed": seed,
                           "n_xxpyy": n_gates, "n_cp": len(rungs),
                           "bp_residual_max": float(max(residuals) if residuals else 0.0)})


CONFIGS = {
    # name: (lattice, chi, chi_env, layers, n_samples, uniform_seed)
    "cfg1": ("square3x3", 4, 16, 2, 1024, 1001),
    "cfg2": ("square6x6", 8, 32, 5, 10000, 1002),
    "cfg3": ("eagle127", 16, 64, 20, 100000, 1003),
    "cfg4a": ("willow105", 32, 128, 7, 100000, 1004),
    "cfg4b": ("willow105", 32, 128, 15, 100000, 1005),
    "P1": ("willow105", 8, 32, 15, 1000, 1008),
    # LUCJ-like (rot_layers brickwork layers before and after the CP layer; 13 + 13 layers
    # give 1300 / 1820 XX+YY rotations on 52 / 72 qubits, "~1800")
    "cfg5a": ("lucj52", 64, 256, 13, 100000, 1006),
    "cfg5b": ("lucj72", 64, 256, 13, 100000, 1007),
}
LUCJ = {"cfg5a": (5, 2006), "cfg5b": (27, 2007)}  # (HF-like occupation per register, circuit seed)


def config_state(name: str, chi: int = None, layers: int = None):
    """The state of a SURVEY 8(d) configuration (optionally at another chi / depth)."""
    lat_name, chi0, _, layers0, _, _ = CONFIGS[name]
    lat = L.by_name(lat_name)
    chi = chi0 if chi is None else chi
    layers = layers0 if layers is None else layers
    if name in LUCJ:
        n_occ, seed = LUCJ[name]
        return lat, lucj_circuit(lat, chi, n_occ, layers, seed)
    return lat, heisenberg_quench(lat, chi, layers)
