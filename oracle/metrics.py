"""ORACLE (test infrastructure only) -- sample-quality metrics of PAPER.md:114-128, 295-300.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.
"""
from __future__ import annotations

import numpy as np


def kld(logq, logp):
    """Sample KLD, Eq. (kld): mean over samples of log q(x)/p(x)."""
    return float(np.mean(np.asarray(logq) - np.asarray(logp)))


def norm_estimate(logq, logp):
    """E_q[p/q] = <psi|psi>: mean ratio and its standard error."""
    r = np.exp(np.asarray(logp) - np.asarray(logq))
    return float(r.mean()), float(r.std(ddof=1) / np.sqrt(len(r))) if len(r) > 1 else 0.0


def importance_expectation(logq, logp, diag_values):
    """(1/N) sum_i (p/q)_i <x_i|O|x_i>, N = mean ratio."""
    r = np.exp(np.asarray(logp) - np.asarray(logq))
    return float(np.sum(r * np.asarray(diag_values)) / np.sum(r))
