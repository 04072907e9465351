"""Processor-shaped graphs and their row partitions (shared, seeded input structure).

This module holds NO arithmetic of the method. It only builds the graphs the paper samples
from and the line partitions ("rows") the boundary-MPS sweep walks through:

* square L_r x L_c lattice, rows = grid rows               (configs 1, 2)
* IBM Eagle-127 heavy-hex in grid coordinates               (config 3, R17)
* Google-Willow-like 105-qubit rotated square lattice       (config 4, P1)
* LUCJ-like two-register ladders (52 / 72 qubits)           (config 5)

Vertex ids are assigned in row order (row 0 first, left to right), so ``rows`` is a list of
consecutive id ranges; callers may relabel vertices to exercise general row orders.
Edge ids are the positions in ``edges``; every edge is stored as (u, v) with u < v.
``colours`` is the Trotter edge colouring of R19 (K groups of
non-overlapping pairs, K = z on bipartite lattices).
The display coordinates are reconstructions (PAPER.md shows the layouts only in figures,
PAPER.md:39, R17) and are used for the domain-wall split (R18).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class Lattice:
    name: str
    n: int
    edges: list          # [(u, v)], u < v, edge id = index
    coords: list         # display (x, y) per vertex
    rows: list           # [[vertex ids in row order]] -- the line partition b = 1..N_b
    colours: list = field(default_factory=list)  # [[edge ids]] per Trotter colour group

    @property
    def n_edges(self) -> int:
        return len(self.edges)

    def degree(self) -> list:
        deg = [0] * self.n
        for u, v in self.edges:
            deg[u] += 1
            deg[v] += 1
        return deg

    def n_loops(self) -> int:
        """Primitive-loop count of a connected planar graph, |E| - |V| + 1 (Euler)."""
        return self.n_edges - self.n + 1


def _bipartite_colouring(n: int, edges: list) -> list:
    """Edge colouring of a bipartite graph with max-degree colours (Koenig's theorem,
    PAPER.md:167), built by the alternating-path method in edge-id order (R19)."""
    deg = [0] * n
    for u, v in edges:
        deg[u] += 1
        deg[v] += 1
    K = max(deg) if deg else 0
    at = [dict() for _ in range(n)]  # vertex -> {colour: edge id}
    col = [-1] * len(edges)

    def free(x):
        for c in range(K):
            if c not in at[x]:
                return c
        raise RuntimeError("no free colour")

    for eid, (u, v) in enumerate(edges):
        a = free(u)
        b = free(v)
        if a not in at[v]:
            c = a
        elif b not in at[u]:
            c = b
        else:
            # flip the a/b alternating path that starts at v with colour a
            path = []
            x, cur = v, a
            while cur in at[x]:
                e = at[x][cur]
                path.append(e)
                p, q = edges[e]
                x = q if p == x else p
                cur = b if cur == a else a
            for e in path:
                p, q = edges[e]
                old = col[e]
                del at[p][old]
                del at[q][old]
            for e in path:
                p, q = edges[e]
                new = b if col[e] == a else a
                col[e] = new
                at[p][new] = e
                at[q][new] = e
            c = a
        col[eid] = c
        at[u][c] = eid
        at[v][c] = eid
    groups = [[] for _ in range(K)]
    for eid, c in enumerate(col):
        groups[c].append(eid)
    return [g for g in groups if g]


def _grid_colouring(edges, pos):
    """R19 for grids: (horizontal, left col even), (horizontal, odd), (vertical, upper row
    even), (vertical, odd); pos[v] = (row, col) in lattice coordinates."""
    groups = [[], [], [], []]
    for eid, (u, v) in enumerate(edges):
        (ru, cu), (rv, cv) = pos[u], pos[v]
        if ru == rv:
            groups[0 if min(cu, cv) % 2 == 0 else 1].append(eid)
        else:
            groups[2 if min(ru, rv) % 2 == 0 else 3].append(eid)
    return [g for g in groups if g]


def _from_points(name, pts, coords):
    """Build a lattice from lattice points (row, col): horizontal edges between consecutive
    columns of a row, vertical edges between equal columns of consecutive rows."""
    pts_sorted = sorted(pts)
    vid = {p: i for i, p in enumerate(pts_sorted)}
    rows = {}
    for (r, c) in pts_sorted:
        rows.setdefault(r, []).append(vid[(r, c)])
    edges = []
    for (r, c) in pts_sorted:
        if (r, c + 1) in vid:
            edges.append((vid[(r, c)], vid[(r, c + 1)]))
    for (r, c) in pts_sorted:
        if (r + 1, c) in vid:
            edges.append((vid[(r, c)], vid[(r + 1, c)]))
    pos = {vid[p]: p for p in pts_sorted}
    disp = [coords[p] for p in pts_sorted]
    lat = Lattice(name, len(pts_sorted), edges, disp, [rows[r] for r in sorted(rows)])
    lat.colours = _grid_colouring(edges, pos)
    return lat


def square(n_rows: int, n_cols: int) -> Lattice:
    """Square lattice; rows = grid rows (configs 1-2)."""
    pts = [(r, c) for r in range(n_rows) for c in range(n_cols)]
    coords = {(r, c): (c, r) for (r, c) in pts}
    return _from_points(f"square{n_rows}x{n_cols}", pts, coords)


def willow105() -> Lattice:
    """Willow-like rotated square lattice (config 4 / P1).

    Chip points (x, y) with 0<=x<=13, 0<=y<=14, x+y even, coupled to diagonal neighbours;
    lattice coordinates (row, col) = ((x-y)/2 + 7, (x+y)/2) turn it into a square lattice
    whose 14 lattice rows (widths 1,3,...,13,14,12,...,2) are the partition.
    """
    pts, coords = [], {}
    for x in range(14):
        for y in range(15):
            if (x + y) % 2 == 0:
                p = ((x - y) // 2 + 7, (x + y) // 2)
                pts.append(p)
                coords[p] = (x, y)
    lat = _from_points("willow105", pts, coords)
    assert lat.n == 105 and lat.n_edges == 182, (lat.n, lat.n_edges)
    return lat


def rotated_patch(nx: int, ny: int) -> Lattice:
    """A small Willow-like rotated square patch: chip points (x, y), 0 <= x < nx, 0 <= y < ny,
    x + y even, diagonal couplings (the willow105 construction on a smaller chip; exact-regime
    tests of the chip-row partition)."""
    pts, coords = [], {}
    for x in range(nx):
        for y in range(ny):
            if (x + y) % 2 == 0:
                p = ((x - y) // 2 + ny // 2, (x + y) // 2)
                pts.append(p)
                coords[p] = (x, y)
    return _from_points(f"rotated{nx}x{ny}", pts, coords)


def chip_rows(lat: Lattice) -> list:
    """The chip-row ("diagonal") partition of a rotated square lattice: rows = chip
    rows y (display coordinates), vertices by x. Every interior vertex has two up and two down
    edges and no edge inside its row (NEXT-3); see tninputs.synthetic.split_two_edge_vertices."""
    rows = {}
    for v, (x, y) in enumerate(lat.coords):
        rows.setdefault(y, []).append(v)
    return [sorted(rows[y], key=lambda v: lat.coords[v][0]) for y in sorted(rows)]


def eagle127() -> Lattice:
    """IBM Eagle heavy-hex in grid coordinates (config 3).

    13 grid rows: long rows 0,2,..,12 (row 0: cols 0-13, rows 2-10: cols 0-14, row 12:
    cols 1-14); bridge rows 1,3,..,11 at cols {0,4,8,12} (rows 1,5,9) or {2,6,10,14}
    (rows 3,7,11). 127 qubits, 144 edges, 18 primitive loops of 12 edges.
    """
    occupied = {}
    for r in range(13):
        if r % 2 == 0:
            cols = range(0, 14) if r == 0 else (range(1, 15) if r == 12 else range(0, 15))
        else:
            cols = (0, 4, 8, 12) if (r // 2) % 2 == 0 else (2, 6, 10, 14)
        occupied[r] = list(cols)
    vid, rows, coords = {}, [], []
    for r in range(13):
        row = []
        for c in occupied[r]:
            vid[(r, c)] = len(coords)
            coords.append((c, r))
            row.append(vid[(r, c)])
        rows.append(row)
    edges = []
    for r in range(0, 13, 2):
        cs = occupied[r]
        for c0, c1 in zip(cs, cs[1:]):
            edges.append((vid[(r, c0)], vid[(r, c1)]))
    for r in range(1, 13, 2):
        for c in occupied[r]:
            edges.append((vid[(r - 1, c)], vid[(r, c)]))
            edges.append((vid[(r, c)], vid[(r + 1, c)]))
    lat = Lattice("eagle127", len(coords), edges, coords, rows)
    lat.colours = _bipartite_colouring(lat.n, edges)
    assert lat.n == 127 and lat.n_edges == 144 and lat.n_loops() == 18
    return lat


def lucj_ladder(n_reg: int, rung_every: int) -> Lattice:
    """LUCJ-like two-register ladder (config 5): alpha and beta chains of
    n_reg qubits, rungs at i = 0 mod rung_every; rows = rung pairs {alpha_i, beta_i}
    (the paper's column partition)."""
    edges, coords, rows = [], [], []
    for i in range(n_reg):
        rows.append([2 * i, 2 * i + 1])
        coords += [(i, 0), (i, 1)]
    for i in range(n_reg - 1):
        edges.append((2 * i, 2 * i + 2))
    for i in range(n_reg - 1):
        edges.append((2 * i + 1, 2 * i + 3))
    for i in range(0, n_reg, rung_every):
        edges.append((2 * i, 2 * i + 1))
    lat = Lattice(f"lucj{2 * n_reg}", 2 * n_reg, edges, coords, rows)
    lat.colours = _bipartite_colouring(lat.n, edges)
    return lat


def chain(n: int) -> Lattice:
    """Path graph, one vertex per row (a line partition of a chain)."""
    edges = [(i, i + 1) for i in range(n - 1)]
    lat = Lattice(f"chain{n}", n, edges, [(i, 0) for i in range(n)], [[i] for i in range(n)])
    lat.colours = [[e for e in range(n - 1) if e % 2 == 0], [e for e in range(n - 1) if e % 2 == 1]]
    lat.colours = [g for g in lat.colours if g]
    return lat


def row_strip(lat: Lattice, b0: int, b1: int) -> Lattice:
    """Rows b0..b1-1 of a lattice as a lattice of its own (vertices renumbered in row order,
    edges among them kept, edge order preserved): a few rows of the full chip at the full
    row widths, for exact-regime tests at the metric tensor shapes."""
    keep = [v for r in lat.rows[b0:b1] for v in r]
    new = {v: i for i, v in enumerate(keep)}
    edges = [(new[u], new[v]) for (u, v) in lat.edges if u in new and v in new]
    edges = [(min(e), max(e)) for e in edges]
    rows = [[new[v] for v in r] for r in lat.rows[b0:b1]]
    out = Lattice(f"{lat.name}_rows{b0}to{b1}", len(keep), edges, [lat.coords[v] for v in keep], rows)
    out.colours = _bipartite_colouring(out.n, edges)
    return out


def by_name(name: str) -> Lattice:
    if name.startswith("square"):
        r, c = name[len("square"):].split("x")
        return square(int(r), int(c))
    if name == "willow105":
        return willow105()
    if name == "eagle127":
        return eagle127()
    if name == "lucj52":
        return lucj_ladder(26, 4)
    if name == "lucj72":
        return lucj_ladder(36, 8)
    if name.startswith("chain"):
        return chain(int(name[len("chain"):]))
    raise ValueError(name)


def domain_wall_bits(lat: Lattice) -> list:
    """R18 (PAPER.md:180 'split the system into two halves'): the first floor(N/2)
    vertices in (display-x, display-y) lexicographic order are |0>, the rest |1>."""
    order = sorted(range(lat.n), key=lambda v: (lat.coords[v][0], lat.coords[v][1], v))
    bits = [1] * lat.n
    for v in order[: lat.n // 2]:
        bits[v] = 0
    return bits


def row_csr(rows: list):
    """(row_ptr, row_vertices) of a row partition, the C-ABI layout."""
    ptr = [0]
    verts = []
    for r in rows:
        verts += list(r)
        ptr.append(len(verts))
    return ptr, verts
