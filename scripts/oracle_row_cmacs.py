"""Per-row complex MACs of one oracle sample (oracle.bmps.sample), counted by bench.py's
shape-only dry run of the oracle's pairwise contractions, and the shapes of each row's
incoming boundary MPS; written to profiles/oracle_row_cmacs.json for the bounded CPU-oracle
timings of bench.py (the oracle times one row and scales by its share of the sample's
work). Calls only oracle/ and tninputs/ (no CUDA path).

python scripts/oracle_row_cmacs.py [workload ...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import bmps as B  # noqa: E402
from tninputs import lattices as L  # noqa: E402

path = os.path.join(ROOT, "profiles", "oracle_row_cmacs.json")
table = json.load(open(path)) if os.path.exists(path) else {}
for wl in sys.argv[1:] or [bench.DEFAULT_WORKLOAD]:
    lat_name, chi, R, _ = bench.WORKLOADS[wl]
    lat = L.by_name(lat_name)
    st = bench.make_state(lat, chi)
    P = B.Prepared(st, lat.rows)
    M = bench.LazyRandomM(P, R, np.random.default_rng(7))
    rc, ms = bench.oracle_dry_run(P, M, R)
    table[wl] = {"row_cmacs": rc, "m_shapes": [None if m is None else [list(t) for t in m] for m in ms]}
    print(wl, f"{sum(rc):.4e} complex MACs per sample", flush=True)
json.dump(table, open(path, "w"), indent=1)
