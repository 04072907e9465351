"""Shared helpers of the GPU parity tests: oracle runs and the R16 tolerance check.

R16 (north star "per-sample conditional probabilities and log p(x) within
1e-4 relative ... bitstrings identical except where a uniform falls within 1e-4 of a CDF
boundary"): conditionals |dP| <= 1e-4 P_ref (+1e-6 absolute floor when P_ref < 1e-2);
ln q: |d| <= 1e-4 max(1, |ln q_ref|); amplitudes |exp(d ln|a| + i d phi) - 1| <= 1e-4.
"""
from __future__ import annotations

import math

import numpy as np

REL = 1e-4
FLOOR = 1e-6
BOUNDARY = 1e-4


def oracle_samples(P, M, R, u, n=None):
    from oracle import bmps as B
    n = u.shape[0] if n is None else n
    bits = np.zeros((n, P.n), np.uint8)
    logq = np.zeros(n)
    cond = np.zeros((n, P.n))
    for k in range(n):
        b, lq, c, _ = B.sample(P, M, R, u[k])
        bits[k], logq[k], cond[k] = b, lq, c
    return bits, logq, cond


def compare_samples(order, u, gbits, glogq, gcond, rbits, rlogq, rcond):
    """Returns a report dict; raises AssertionError on a tolerance violation."""
    n = gbits.shape[0]
    boundary = 0
    worst_rel = 0.0
    compared = 0
    for k in range(n):
        diverged = False
        for v in order:
            pr, pg = rcond[k, v], gcond[k, v]
            if gbits[k, v] != rbits[k, v]:
                p0 = pr if rbits[k, v] == 0 else 1 - pr
                assert abs(u[k, v] - p0) < BOUNDARY, (k, v, u[k, v], p0)
                boundary += 1
                diverged = True
                break
            tol = REL * pr + (FLOOR if pr < 1e-2 else 0.0)
            assert abs(pg - pr) <= tol, (k, v, pg, pr)
            if pr > 0:
                worst_rel = max(worst_rel, abs(pg - pr) / pr)
            compared += 1
        if not diverged:
            assert abs(glogq[k] - rlogq[k]) <= REL * max(1.0, abs(rlogq[k])), (k, glogq[k], rlogq[k])
    return {"boundary": boundary, "worst_rel": worst_rel, "compared": compared}


def amp_close(la_g, ph_g, la_r, ph_r, zero_by_symmetry=False, log_scale=None):
    """R16 for amplitudes: |exp(d ln|a| + i d phi) - 1| <= 1e-4.

    zero_by_symmetry: the bitstring lies outside the state's U(1) magnetisation sector
    (the Heisenberg quench conserves the magnetisation of the domain wall), so
    <x|psi> = 0 exactly and only round-off remains on either side; no relative comparison
    exists, and the GPU value must be negligible: below 1e-4 of sqrt(<psi|psi>)
    (log_scale = ln sqrt(<psi|psi>)). Every other amplitude takes the relative test."""
    if zero_by_symmetry:
        return math.isinf(la_g) or la_g < log_scale + math.log(1e-4)
    z = np.exp((la_g - la_r) + 1j * (ph_g - ph_r))
    return abs(z - 1) <= REL
