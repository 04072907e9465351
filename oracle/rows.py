"""ORACLE (test infrastructure only) -- row-partition analysis of a TNS.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this
package. Shares no code with paper_2507_11424_b200/.

A line partition ("grouping of the tensors into partitions ... forms a line";
PAPER.md:275) is accepted in the grid-layered form of SURVEY R1: every vertex has at most
one edge to the previous row (up) and one to the next row (down), intra-row edges join
consecutive vertices of a row, and inter-row edges do not cross.
"""
from __future__ import annotations

import numpy as np


class RowError(ValueError):
    pass


def analyse(n, edges, bond_dims, rows):
    """Return per-vertex (b, j, up, down, left, right) edge ids (-1 = absent).

    Raises RowError on anything that is not a grid-layered line partition (R1)."""
    flat = [v for r in rows for v in r]
    if sorted(flat) != list(range(n)) or any(len(r) == 0 for r in rows):
        raise RowError("row order is not a permutation of the vertices")
    pos = {}
    for b, r in enumerate(rows):
        for j, v in enumerate(r):
            pos[v] = (b, j)
    info = {v: {"b": pos[v][0], "j": pos[v][1], "up": -1, "down": -1, "left": -1, "right": -1}
            for v in range(n)}
    for e, (u, v) in enumerate(edges):
        (bu, ju), (bv, jv) = pos[u], pos[v]
        if bu == bv:
            if abs(ju - jv) != 1:
                raise RowError(f"intra-row edge {e} joins non-consecutive vertices")
            a, c = (u, v) if ju < jv else (v, u)
            if info[a]["right"] != -1 or info[c]["left"] != -1:
                raise RowError("duplicate intra-row edge")
            info[a]["right"] = e
            info[c]["left"] = e
        elif abs(bu - bv) == 1:
            a, c = (u, v) if bu < bv else (v, u)
            if info[a]["down"] != -1 or info[c]["up"] != -1:
                raise RowError(f"vertex with more than one up/down edge (edge {e})")
            info[a]["down"] = e
            info[c]["up"] = e
        else:
            raise RowError(f"edge {e} skips a row")
    for b in range(len(rows) - 1):
        pairs = []
        for v in rows[b]:
            e = info[v]["down"]
            if e >= 0:
                u, w = edges[e]
                other = w if u == v else u
                pairs.append((info[v]["j"], info[other]["j"]))
        pairs.sort()
        lows = [p[1] for p in pairs]
        if any(x >= y for x, y in zip(lows, lows[1:])):
            raise RowError(f"crossing inter-row edges between rows {b} and {b + 1}")
    return info


def site_tensors(state, rows):
    """A_v[s, u, d, l, r] (missing legs of dim 1) from the file layout (2, d_e1, ...),
    e1 < e2 < ...."""
    n = state["n"]
    edges = [tuple(e) for e in np.asarray(state["edges"]).tolist()]
    info = analyse(n, edges, state["bond_dims"], rows)
    inc = [[] for _ in range(n)]
    for e, (u, v) in enumerate(edges):
        inc[u].append(e)
        inc[v].append(e)
    A = []
    for v in range(n):
        t = np.asarray(state["tensors"][v], dtype=np.complex128)
        legs = inc[v]
        order = [0]
        shape = [2]
        for key in ("up", "down", "left", "right"):
            e = info[v][key]
            if e >= 0:
                order.append(1 + legs.index(e))
        t = np.transpose(t, order)
        full = [2]
        for key in ("up", "down", "left", "right"):
            e = info[v][key]
            full.append(int(state["bond_dims"][e]) if e >= 0 else 1)
        A.append(t.reshape(full))
    return A, info
