"""Enumeration oracle: every support of size <= k, each
box-constrained ridge / logistic restriction solved to ~1e-10.  numpy/scipy only;
test infrastructure.
"""
import itertools
import math

import numpy as np
from scipy.optimize import minimize


def _sq_box_ridge(XS, y, lam, M):
    """min 1/2|y - XS b|^2 + lam |b|^2, |b|_inf <= M: exact active-set enumeration."""
    q = XS.shape[1]
    if q == 0:
        return 0.5 * float(y @ y), np.zeros(0)
    H = XS.T @ XS + 2 * lam * np.eye(q)
    g = XS.T @ y
    best = (math.inf, None)
    for pattern in itertools.product((0, 1, -1), repeat=q):  # 0 free, +-1 at +-M
        pat = np.array(pattern)
        free = pat == 0
        b = np.where(free, 0.0, pat * M)
        if free.any():
            rhs = g[free] - H[np.ix_(free, ~free)] @ b[~free]
            b[free] = np.linalg.solve(H[np.ix_(free, free)], rhs)
            if np.any(np.abs(b[free]) > M + 1e-12):
                continue
        grad = H @ b - g
        ok = True
        for j in range(q):  # KKT at the bounds
            if pat[j] == 1 and grad[j] > 1e-9:
                ok = False
            if pat[j] == -1 and grad[j] < -1e-9:
                ok = False
        if not ok:
            continue
        r = y - XS @ b
        f = 0.5 * float(r @ r) + lam * float(b @ b)
        if f < best[0]:
            best = (f, b)
    return best


def _logistic_box_ridge(XS, y, lam, M):
    q = XS.shape[1]
    n = len(y)
    if q == 0:
        return n * math.log(2.0), np.zeros(0)

    def fg(b):
        t = -y * (XS @ b)
        f = np.sum(np.logaddexp(0.0, t)) + lam * b @ b
        sig = np.exp(-np.logaddexp(0.0, -t))  # sigmoid(t)
        grad = XS.T @ (-y * sig) + 2 * lam * b
        return f, grad

    res = minimize(fg, np.zeros(q), jac=True, method="L-BFGS-B", bounds=[(-M, M)] * q,
                   options=dict(ftol=1e-15, gtol=1e-11, maxiter=10000))
    return float(res.fun), res.x


def all_support_values(X, y, loss, k, M, lam):
    """{sorted support tuple: v(S)} for every |S| <= k."""
    p = X.shape[1]
    vals = {}
    for q in range(0, k + 1):
        for S in itertools.combinations(range(p), q):
            XS = X[:, list(S)]
            if loss == 0:
                f, _ = _sq_box_ridge(XS, y, lam, M)
            else:
                f, _ = _logistic_box_ridge(XS, y, lam, M)
            vals[S] = f
    return vals


def node_optimum(vals, j0, j1):
    z, o = set(j0), set(j1)
    best = math.inf
    for S, f in vals.items():
        s = set(S)
        if o <= s and not (s & z):
            best = min(best, f)
    return best
