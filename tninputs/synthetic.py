"""Seeded synthetic tensor-network states and uniforms (shared input generators).

Holds no arithmetic of the sampling method (no fits, environments, conditionals). It only
builds input states in the interchange layout of the C-ABI:

    tensors[v] : complex128, C-order shape (2, d_e1, d_e2, ...) where e1 < e2 < ... are
                 the ids of the edges incident to v (physical index first).

Generators
* ``vidal_like``  -- dense random tensors with singular-value-weighted bonds, the value
  distribution of simple-update outputs in Vidal/BP gauge (SURVEY 8(d)
  "Value distribution"). Used for the throughput workload.
* ``branch_superposition`` -- |psi> = sum_c prod_v phi_v^(c), embedded at bond dimension
  chi with dense bi-orthogonal leg vectors, so every boundary has exact rank <= K (single
  layer) / K^2 (double layer) while all tensors are dense at full shape. Its q(x) and
  conditionals have a closed form (full-scale pin, SURVEY 8(c.4) "product state embedded
  at bond dim chi", generalised to K branches; K=1 is the gauged product state, K=2 with
  basis branches is GHZ).
* ``product_state`` -- bond dimension 1 (PAPER.md:180 initial state).
* ``uniforms`` -- numpy default_rng(seed).random((n, N)) float64.
"""
from __future__ import annotations

import numpy as np


def incident_edges(n: int, edges) -> list:
    inc = [[] for _ in range(n)]
    for eid, (u, v) in enumerate(edges):
        inc[u].append(eid)
        inc[v].append(eid)
    return inc


def make_state(lat, tensors, bond_dims, chi, meta=None) -> dict:
    return {
        "n": lat.n,
        "edges": np.asarray(lat.edges, dtype=np.int32).reshape(-1, 2),
        "bond_dims": np.asarray(bond_dims, dtype=np.int32),
        "chi": int(chi),
        "tensors": [np.ascontiguousarray(t, dtype=np.complex128) for t in tensors],
        "meta": dict(meta or {}),
    }


def uniforms(n_samples: int, n_vertices: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).random((n_samples, n_vertices))


def product_state(lat, bits) -> dict:
    inc = incident_edges(lat.n, lat.edges)
    tensors = []
    for v in range(lat.n):
        t = np.zeros((2,) + (1,) * len(inc[v]), dtype=np.complex128)
        t[(bits[v],) + (0,) * len(inc[v])] = 1.0
        tensors.append(t)
    return make_state(lat, tensors, [1] * lat.n_edges, 1, {"kind": "product", "bits": list(bits)})


def _cgauss(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def vidal_like(lat, chi: int, seed: int, xi: float = 8.0) -> dict:
    """A_v = Gamma_v x prod_e sqrt(lambda_e) with Gamma_v complex Gaussian and a decaying
    bond spectrum lambda_e[k] ~ exp(-k / xi) (normalised): the dense, singular-value-
    weighted tensors a BP-gauged simple update produces. Every bond at chi
    (the memory upper bound of SURVEY 6)."""
    rng = np.random.default_rng(seed)
    inc = incident_edges(lat.n, lat.edges)
    lam = []
    for _ in lat.edges:
        s = np.exp(-np.arange(chi) / xi) * np.exp(0.1 * rng.standard_normal(chi))
        s = np.sort(s)[::-1]
        lam.append(s / np.linalg.norm(s))
    tensors = []
    for v in range(lat.n):
        shape = (2,) + (chi,) * len(inc[v])
        t = _cgauss(rng, shape)
        for ax, e in enumerate(inc[v]):
            w = np.sqrt(lam[e]).reshape([-1 if i == ax + 1 else 1 for i in range(len(shape))])
            t = t * w
        t /= np.linalg.norm(t)
        tensors.append(t)
    return make_state(lat, tensors, [chi] * lat.n_edges, chi,
                      {"kind": "vidal_like", "seed": seed, "xi": xi})


def branch_superposition(lat, chi: int, K: int, seed: int, phis=None, gauge: bool = True) -> dict:
    """|psi> = sum_{c<K} prod_v phi_v^(c)  at bond dimension chi (requires K <= chi).

    On each edge e=(v,w) pick V_e (K x chi) and W_e (chi x K) with V_e W_e = I_K; the leg
    vectors a_{v,e}^(c) = V_e[c], a_{w,e}^(c) = W_e[:, c] then contract to delta_{cc'} along
    e, so the network equals the branch sum exactly (no arithmetic of the method).
    phis: array (K, N, 2) complex, default random.  Returns the state with meta['phis'].
    """
    assert 1 <= K <= chi
    rng = np.random.default_rng(seed)
    inc = incident_edges(lat.n, lat.edges)
    if phis is None:
        phis = _cgauss(rng, (K, lat.n, 2))
    phis = np.asarray(phis, dtype=np.complex128)
    legs = {}
    for e, (u, w) in enumerate(lat.edges):
        V = _cgauss(rng, (K, chi)) / np.sqrt(chi)
        W = V.conj().T @ np.linalg.inv(V @ V.conj().T)
        if gauge and chi > K:
            Z = _cgauss(rng, (chi, K)) / np.sqrt(chi)
            W = W + (np.eye(chi) - W @ V) @ Z
        legs[(u, e)] = V            # rows: a_{u,e}^(c)
        legs[(w, e)] = W.T          # rows: a_{w,e}^(c)
    tensors = []
    for v in range(lat.n):
        shape = (2,) + (chi,) * len(inc[v])
        t = np.zeros(shape, dtype=np.complex128)
        for c in range(K):
            term = phis[c, v]
            for e in inc[v]:
                term = np.multiply.outer(term, legs[(v, e)][c])
            t += term
        tensors.append(t)
    return make_state(lat, tensors, [chi] * lat.n_edges, chi,
                      {"kind": "branch_superposition", "K": K, "seed": seed, "phis": phis})


def ghz(lat, chi: int = 2, seed: int = 0) -> dict:
    """GHZ (|0..0> + |1..1>) embedded at bond dimension chi."""
    phis = np.zeros((2, lat.n, 2), dtype=np.complex128)
    phis[0, :, 0] = 1.0
    phis[1, :, 1] = 1.0
    st = branch_superposition(lat, chi, 2, seed, phis=phis, gauge=chi > 2)
    st["meta"]["kind"] = "ghz"
    return st


def save_state(path, st) -> None:
    arrs = {
        "n": np.int64(st["n"]),
        "edges": st["edges"],
        "bond_dims": st["bond_dims"],
        "chi": np.int64(st["chi"]),
    }
    for v, t in enumerate(st["tensors"]):
        arrs[f"t{v}"] = t
    for k, val in st.get("meta", {}).items():
        arrs[f"meta_{k}"] = np.asarray(val)
    np.savez(path, **arrs)


def load_state(path) -> dict:
    z = np.load(path, allow_pickle=False)
    n = int(z["n"])
    meta = {k[5:]: z[k] for k in z.files if k.startswith("meta_")}
    return {
        "n": n,
        "edges": z["edges"],
        "bond_dims": z["bond_dims"],
        "chi": int(z["chi"]),
        "tensors": [z[f"t{v}"] for v in range(n)],
        "meta": meta,
    }


def relabel(st: dict, rows: list, perm: list):
    """Relabel vertex v -> perm[v] (and permute tensor legs to keep edge-id order).
    Returns (state, rows) -- exercises general row orders through the C-ABI."""
    n = st["n"]
    edges = [(perm[u], perm[v]) for (u, v) in st["edges"].tolist()]
    order = sorted(range(len(edges)), key=lambda e: (min(edges[e]), max(edges[e])))
    new_edges = [tuple(sorted(edges[e])) for e in order]
    new_bd = [int(st["bond_dims"][e]) for e in order]
    old_of_new = {new: old for new, old in enumerate(order)}
    inc_old = incident_edges(n, st["edges"].tolist())
    inc_new = incident_edges(n, new_edges)
    tensors = [None] * n
    for v in range(n):
        w = perm[v]
        # new leg order: edges incident to w sorted by new id; map back to old positions
        old_pos = [inc_old[v].index(old_of_new[e]) for e in inc_new[w]]
        tensors[w] = np.transpose(st["tensors"][v], [0] + [p + 1 for p in old_pos])
    new_rows = [[perm[v] for v in r] for r in rows]
    out = dict(st)
    out["edges"] = np.asarray(new_edges, dtype=np.int32).reshape(-1, 2)
    out["bond_dims"] = np.asarray(new_bd, dtype=np.int32)
    out["tensors"] = [np.ascontiguousarray(t) for t in tensors]
    return out, new_rows


def split_two_edge_vertices(st: dict, rows: list, xcoord) -> tuple:
    """Rewrite a TNS so that a partition whose vertices have two up or two down edges (the
    chip-row / "diagonal" partition of the Willow layout, NEXT-3) becomes a
    line partition with at most one up and one down edge per vertex (R1). Pure re-indexing, no
    arithmetic of the method: a vertex v with two up or two down edges is replaced by
      L_v[s, left edges..., k] = delta(s, 0) delta(k, (left edges))   (no qubit: s = 1 slice zero)
      R_v[s, right edges..., k] = A_v[s, all edges]                   (the qubit, keeps id v)
    joined by a new edge k of dimension prod(left edge dims); 'left' edges are those whose other
    end has a smaller xcoord. In the row, v becomes (L_v, v). The boundary between two rows then has
    one site per crossing edge, as in the paper's diagonal contraction. L_v's drawn bit is always
    0 with conditional 1 (its s = 1 slice vanishes), so q(x) and the qubits' bits are unchanged.

    Returns (state, rows, n_qubits): vertex ids < n_qubits are the original qubits."""
    n = st["n"]
    edges = [tuple(int(a) for a in e) for e in np.asarray(st["edges"]).reshape(-1, 2).tolist()]
    bd = [int(d) for d in st["bond_dims"]]
    row_of = {v: b for b, r in enumerate(rows) for v in r}
    inc = incident_edges(n, edges)
    new_edges, new_bd = list(edges), list(bd)
    tensors = [np.asarray(t) for t in st["tensors"]]
    new_tensors = list(tensors)
    new_rows = [list(r) for r in rows]
    next_id = n
    for v in range(n):
        b = row_of[v]
        ups = [e for e in inc[v] if row_of[edges[e][0] + edges[e][1] - v] == b - 1]
        downs = [e for e in inc[v] if row_of[edges[e][0] + edges[e][1] - v] == b + 1]
        if len(ups) < 2 and len(downs) < 2:
            continue
        assert all(row_of[edges[e][0] + edges[e][1] - v] != b for e in inc[v]), "intra-row edge at a split vertex"
        left = [e for e in inc[v] if xcoord[edges[e][0] + edges[e][1] - v] < xcoord[v]]
        right = [e for e in inc[v] if e not in left]
        lv = next_id
        next_id += 1
        ke = len(new_edges)
        kdim = int(np.prod([bd[e] for e in left])) if left else 1
        new_edges.append((lv, v))
        new_bd.append(kdim)
        for e in left:  # the left edges now end at L_v
            u = edges[e][0] + edges[e][1] - v
            new_edges[e] = (u, lv)
        # L_v: axes (s, left edges in id order, k)
        lt = np.zeros((2,) + tuple(bd[e] for e in left) + (kdim,), dtype=np.complex128)
        lt[0] = np.eye(kdim, dtype=np.complex128).reshape(tuple(bd[e] for e in left) + (kdim,))
        # R_v: A_v with the left legs fused into k, axes (s, right edges in id order, k)
        a = tensors[v]
        pos = {e: 1 + i for i, e in enumerate(inc[v])}
        perm = [0] + [pos[e] for e in right] + [pos[e] for e in left]
        rt = np.transpose(a, perm).reshape((2,) + tuple(bd[e] for e in right) + (kdim,))
        new_tensors[v] = np.ascontiguousarray(rt)
        new_tensors.append(np.ascontiguousarray(lt))
        r = new_rows[b]
        r.insert(r.index(v), lv)
    # relabel edges so that (u, v) has u < v; tensors keep legs in increasing edge id, which
    # holds because the new edge k has the largest id at both of its ends
    out_edges = [(min(u, w), max(u, w)) for (u, w) in new_edges]
    out = dict(st)
    out["n"] = next_id
    out["edges"] = np.asarray(out_edges, dtype=np.int32).reshape(-1, 2)
    out["bond_dims"] = np.asarray(new_bd, dtype=np.int32)
    out["chi"] = int(max([int(st["chi"])] + new_bd))
    out["tensors"] = new_tensors
    out["meta"] = dict(st.get("meta", {}), split_from=n)
    return out, new_rows, n
