#!/usr/bin/env python
"""Write oracle goldens for the GPU parity tests (calls only oracle/ and tninputs/).

  python scripts/make_golden.py p1     # P1: Willow-105 L=15 domain-wall quench, chi=8, chi_env=32
  python scripts/make_golden.py w16    # Willow-105 Vidal-like state, chi=16, chi_env=64
  python scripts/make_golden.py cfg3   # config 3: Eagle-127 L=20 quench, chi=16, chi_env=64

Every stored value comes from the CPU oracle (oracle/bmps.py, complex128) on seeded inputs;
nothing is read from the CUDA path. P1's state (SURVEY 8(d) "P1 (parity aux)") is the
oracle generator's quench (oracle/generator.py) rounded to complex64 so
that the file stays small; that rounded state IS the P1 input of both sides (the oracle
below samples from exactly the stored tensors).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import bmps as B  # noqa: E402
from oracle import generator as G  # noqa: E402
from tninputs import lattices as L  # noqa: E402
from tninputs import synthetic as S  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

CASES = {
    # name: (state recipe, chi, chi_env, n samples, uniform seed)
    "p1": ("quench", 8, 32, 64, 1008),
    "w16": ("vidal_like", 16, 64, 8, 1016),
    "cfg3": ("quench", 16, 64, 24, 1003),
}


def state_for(name):
    recipe, chi, *_ = CASES[name]
    cfg = {"p1": "P1", "cfg3": "cfg3"}.get(name)
    lat = L.by_name(G.CONFIGS[cfg][0]) if cfg else L.willow105()
    if recipe == "quench":
        path = os.path.join(GOLDEN, f"{name}_state.npz")
        if os.path.exists(path):
            return lat, load_p1_state(path)
        layers = G.CONFIGS[cfg][3]
        st = G.heisenberg_quench(lat, chi, layers)
        st["tensors"] = [t.astype(np.complex64).astype(np.complex128) for t in st["tensors"]]
        meta = {k: v for k, v in st["meta"].items() if np.ndim(v) == 0}
        st["meta"] = dict(meta, rounded_to="complex64")
        S.save_state(path, st)
        z = dict(np.load(path))  # stored as complex64 (exact: the state is rounded to complex64)
        np.savez_compressed(path, **{k: (v.astype(np.complex64) if v.dtype == np.complex128 else v) for k, v in z.items()})
        return lat, load_p1_state(path)
    return lat, S.vidal_like(lat, chi, seed=2507)


def load_p1_state(path):
    st = S.load_state(path)
    st["tensors"] = [np.asarray(t, dtype=np.complex128) for t in st["tensors"]]
    return st


def main(name):
    _, chi, R, n, useed = CASES[name]
    t0 = time.time()
    lat, st = state_for(name)
    print(f"[{name}] state {time.time() - t0:.0f} s", flush=True)
    P = B.Prepared(st, lat.rows)
    t0 = time.time()
    M, logs = B.norm_envs(P, R)
    print(f"[{name}] oracle norm environments {time.time() - t0:.0f} s", flush=True)
    u = S.uniforms(n, lat.n, useed)
    bits = np.zeros((n, lat.n), np.uint8)
    logq = np.zeros(n)
    cond = np.zeros((n, lat.n))
    flags = np.zeros(n, np.uint32)
    t0 = time.time()
    for k in range(n):
        bits[k], logq[k], cond[k], flags[k] = B.sample(P, M, R, u[k])
        print(f"[{name}] sample {k} {time.time() - t0:.0f} s", flush=True)
    out = os.path.join(GOLDEN, f"{name}_oracle.npz")
    np.savez_compressed(out, chi=chi, chi_env=R, uniform_seed=useed, bits=bits, logq=logq, cond=cond, flags=flags,
                        log_norm=B.log_norm(P, M, logs))
    print(f"[{name}] wrote {out}", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm)
