"""GPU TNS construction driver: circuits of two-qubit gates applied by the
BP-gauged simple update of libtnsample (tn_su_*, complex FP64 on the device), PAPER.md:65-80,
147-185, 305-322. Argument marshalling and the circuit schedule only: every BP sweep, gauge,
decomposition and truncation runs in the library's kernels.

The circuits are those of the paper's workloads: the domain-wall Heisenberg
quench (first-order Trotter layers over the lattice's colour groups, BP refreshed before every
group) and the synthetic LUCJ-like circuit (XX+YY brickwork, CP on the
rungs, HF-like start). The gate matrices are the closed forms of R22.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import _check, lib


def heisenberg_gate(J: float, dt: float) -> np.ndarray:
    """exp(-i J dt (XX+YY+ZZ)) = e^{i th}[cos 2th I - i sin 2th SWAP], th = J dt (R22)."""
    th = J * dt
    swap = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)
    return np.exp(1j * th) * (np.cos(2 * th) * np.eye(4) - 1j * np.sin(2 * th) * swap)


def xxpyy_gate(theta: float) -> np.ndarray:
    """XX+YY(theta) = exp(-i theta/4 (XX+YY)) (R22)."""
    c, s = np.cos(theta / 2), np.sin(theta / 2)
    return np.array([[1, 0, 0, 0], [0, c, -1j * s, 0], [0, -1j * s, c, 0], [0, 0, 0, 1]], dtype=np.complex128)


def cphase_gate(phi: float) -> np.ndarray:
    return np.diag([1, 1, 1, np.exp(1j * phi)]).astype(np.complex128)


def _su_check(rc):
    if rc != 0:
        from ._lib import TNError
        raise TNError(rc, lib().tn_su_last_error().decode())


class GPUTNS:
    """A TNS under construction on the current CUDA device (tn_su_create)."""

    def __init__(self, lat, bits):
        self.lat = lat
        self.n = lat.n
        self.edges = np.ascontiguousarray(np.asarray(lat.edges, dtype=np.int32).reshape(-1, 2))
        b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8))
        h = C.c_void_p()
        _su_check(lib().tn_su_create(self.n, len(self.edges), self.edges.ctypes.data, b.ctypes.data, C.byref(h)))
        self._h = h
        self.eps = []
        self.residuals = []

    def close(self):
        if getattr(self, "_h", None):
            lib().tn_su_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bp(self, tol=1e-10, max_sweeps=50):
        res = C.c_double()
        sw = C.c_int32()
        _su_check(lib().tn_su_bp(self._h, float(tol), int(max_sweeps), C.byref(res), C.byref(sw)))
        self.residuals.append(res.value)
        return res.value

    def apply2(self, e, G, chi, cutoff=1e-14):
        g = np.ascontiguousarray(np.asarray(G, dtype=np.complex128).reshape(4, 4))
        eps = C.c_double()
        _su_check(lib().tn_su_apply2(self._h, int(e), g.ctypes.data, int(chi), float(cutoff), C.byref(eps)))
        self.eps.append(eps.value)
        return eps.value

    def bond_dims(self):
        out = np.zeros(len(self.edges), dtype=np.int32)
        _su_check(lib().tn_su_bond_dims(self._h, out.ctypes.data))
        return out

    def state(self, chi, meta=None) -> dict:
        dims = self.bond_dims()
        inc = [[] for _ in range(self.n)]
        for e, (u, v) in enumerate(self.edges.tolist()):
            inc[u].append(e)
            inc[v].append(e)
        tensors = [np.zeros((2,) + tuple(int(dims[e]) for e in inc[v]), dtype=np.complex128) for v in range(self.n)]
        ptrs = (C.c_void_p * self.n)(*[t.ctypes.data for t in tensors])
        _su_check(lib().tn_su_export(self._h, ptrs))
        m = dict(meta or {})
        m.update({"eps": np.asarray(self.eps), "fidelity": float(np.prod([1 - x for x in self.eps])),
                  "constructed_on": "gpu"})
        return {"n": self.n, "edges": self.edges.copy(), "bond_dims": dims.astype(np.int32), "chi": int(chi),
                "tensors": tensors, "meta": m}


def heisenberg_quench(lat, bits, chi: int, layers: int, J: float = 1.0, dt: float = 0.1) -> dict:
    """Domain-wall quench on the GPU: L Trotter layers over the lattice's
    colour groups, BP refresh before each group."""
    tns = GPUTNS(lat, bits)
    G = heisenberg_gate(J, dt)
    for _ in range(layers):
        for group in lat.colours:
            tns.bp()
            for e in group:
                tns.apply2(e, G, chi)
    return tns.state(chi, {"kind": "heisenberg", "layers": layers, "J": J, "dt": dt,
                           "bp_residual_max": float(max(tns.residuals) if tns.residuals else 0.0)})
