"""ORACLE (test infrastructure only) -- brute-force statevector of a small TNS (O8).

Contracts every tensor exactly (no truncation), so <x|psi> is the plain definition of the
amplitude network. Basis index = sum_v x_v 2^(N-1-v): vertex 0 is the most
significant bit. Only for N <= ~22.
"""
from __future__ import annotations

import numpy as np


def statevector(state) -> np.ndarray:
    n = state["n"]
    edges = [tuple(e) for e in np.asarray(state["edges"]).tolist()]
    inc = [[] for _ in range(n)]
    for e, (u, v) in enumerate(edges):
        inc[u].append(e)
        inc[v].append(e)
    # running tensor: axes = [phys of vertices 0..v] + [open edge ids]
    psi = np.asarray(state["tensors"][0], dtype=np.complex128)
    open_edges = list(inc[0])
    nphys = 1
    for v in range(1, n):
        t = np.asarray(state["tensors"][v], dtype=np.complex128)
        shared = [e for e in inc[v] if e in open_edges]
        ax_psi = [nphys + open_edges.index(e) for e in shared]
        ax_t = [1 + inc[v].index(e) for e in shared]
        psi = np.tensordot(psi, t, axes=(ax_psi, ax_t))
        # axes now: phys(0..v-1), remaining open edges of psi, phys v, remaining legs of t
        rem_psi = [e for e in open_edges if e not in shared]
        rem_t = [e for e in inc[v] if e not in shared]
        k = len(rem_psi)
        order = list(range(nphys)) + [nphys + k] + [nphys + i for i in range(k)] + \
            [nphys + k + 1 + i for i in range(len(rem_t))]
        psi = np.transpose(psi, order)
        nphys += 1
        open_edges = rem_psi + rem_t
    assert not open_edges
    return psi.reshape(-1)


def bits_of(index: int, n: int):
    return [(index >> (n - 1 - v)) & 1 for v in range(n)]


def conditionals(psi: np.ndarray, n: int, order, bits):
    """Exact sequential conditionals q(x_v | x of earlier vertices in `order`) of the
    normalised distribution |psi(x)|^2 / <psi|psi>; returns the list of
    P(x_v = bits[v] | past) in `order`."""
    p = (np.abs(psi) ** 2).reshape([2] * n)
    p = p / p.sum()
    out = []
    fixed = {}
    for v in order:
        # marginal over all vertices not yet fixed, except v
        idx = [slice(None)] * n
        for w, x in fixed.items():
            idx[w] = x
        sub = p[tuple(idx)]
        free = [w for w in range(n) if w not in fixed]
        axis = free.index(v)
        other = tuple(i for i in range(len(free)) if i != axis)
        marg = sub.sum(axis=other) if other else sub
        tot = marg.sum()
        out.append(marg[bits[v]] / tot)
        fixed[v] = bits[v]
    return out
