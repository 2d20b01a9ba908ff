"""Brute-force active-set solver for Eq. 2 on tiny instances -- a pin for the oracle.

SPEC S:500-508 (``oracle_active_set``): enumerate all 3^m assignments of each variable to
{lower (0), upper (C), free}; for each, solve the equality-constrained linear system on the free
block with the y'a = 0 multiplier, check primal feasibility and the KKT signs at the bounds, and
return the feasible KKT point with the minimum objective.  It belongs to a different algorithm
family than the SMO oracle, so agreement is independent evidence.  Pure numpy; m <= 8.
"""
from __future__ import annotations

import itertools

import numpy as np


def objective(Q, p, a):
    return 0.5 * a @ Q @ a + p @ a


def solve(Q, p, y, C, feas_tol=1e-9):
    Q = np.asarray(Q, np.float64)
    p = np.asarray(p, np.float64)
    y = np.asarray(y, np.float64)
    m = len(p)
    assert m <= 10
    best, best_obj = None, np.inf
    for assign in itertools.product((0, 1, 2), repeat=m):   # 0 lower, 1 upper, 2 free
        a = np.zeros(m)
        F = [i for i in range(m) if assign[i] == 2]
        B = [i for i in range(m) if assign[i] != 2]
        for i in B:
            a[i] = C if assign[i] == 1 else 0.0
        if F:
            nf = len(F)
            K = np.zeros((nf + 1, nf + 1))
            K[:nf, :nf] = Q[np.ix_(F, F)]
            K[:nf, nf] = y[F]
            K[nf, :nf] = y[F]
            rhs = np.zeros(nf + 1)
            rhs[:nf] = -p[F] - (Q[np.ix_(F, B)] @ a[B] if B else 0.0)
            rhs[nf] = -(y[B] @ a[B] if B else 0.0)
            sol, *_ = np.linalg.lstsq(K, rhs, rcond=None)
            if np.abs(K @ sol - rhs).max() > 1e-8:
                continue
            a[F] = sol[:nf]
            lam = sol[nf]
            if (a[F] < -feas_tol).any() or (a[F] > C + feas_tol).any():
                continue
            a[F] = np.clip(a[F], 0.0, C)
            g = Q @ a + p + lam * y
            ok = all(g[i] >= -1e-8 for i in B if assign[i] == 0) and \
                all(g[i] <= 1e-8 for i in B if assign[i] == 1)
            if not ok:
                continue
        else:
            if abs(y @ a) > 1e-12 * max(1.0, C):
                continue
            g = Q @ a + p
            # need lam with g_i + lam y_i >= 0 at lower, <= 0 at upper
            lo, hi = -np.inf, np.inf
            for i in range(m):
                if assign[i] == 0:      # g_i + lam y_i >= 0
                    if y[i] > 0:
                        lo = max(lo, -g[i])
                    else:
                        hi = min(hi, g[i])
                else:                   # g_i + lam y_i <= 0
                    if y[i] > 0:
                        hi = min(hi, -g[i])
                    else:
                        lo = max(lo, g[i])
            if lo > hi + 1e-8:
                continue
        obj = objective(Q, p, a)
        if obj < best_obj:
            best, best_obj = a.copy(), obj
    assert best is not None, "no KKT point: the feasible set contains a = 0, so this is a bug"
    return best, best_obj
