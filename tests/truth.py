"""Ground truth independent of the PDHG method: brute-force vertex enumeration
(acceptance #1) and HiGHS via scipy (a library LP solver).  Used
only to pin the oracle (and, through it, the GPU path) to the plain definition
of the LP optimum, Eq. (1)."""
from __future__ import annotations

import itertools

import numpy as np


def vertex_enumeration(lp) -> float:
    """min c'x over {Gx >= h, Ax = b, l <= x <= u} (all bounds finite) by
    enumerating every basic solution: the m2 equalities plus n - m2 active
    constraints drawn from the >= rows and the 2n bound constraints."""
    K = lp.dense_K()
    n, m1 = lp.n, lp.m1
    G, A = K[:m1], K[m1:]
    h, b = lp.q[:m1], lp.q[m1:]
    assert np.all(np.isfinite(lp.l)) and np.all(np.isfinite(lp.u))
    rows, rhs = [], []
    for i in range(m1):
        rows.append(G[i]); rhs.append(h[i])
    for j in range(n):
        e = np.zeros(n); e[j] = 1.0
        rows.append(e); rhs.append(lp.l[j])
        rows.append(e); rhs.append(lp.u[j])
    rows, rhs = np.array(rows), np.array(rhs)
    best = np.inf
    need = n - A.shape[0]
    for S in itertools.combinations(range(len(rows)), need):
        M = np.vstack([A, rows[list(S)]]) if need else A
        r = np.concatenate([b, rhs[list(S)]]) if need else b
        if np.linalg.matrix_rank(M) < n:
            continue
        x = np.linalg.solve(M, r)
        tol = 1e-9 * (1 + np.abs(x).max())
        if np.all(G @ x >= h - tol) and np.allclose(A @ x, b, atol=tol) and \
                np.all(x >= lp.l - tol) and np.all(x <= lp.u + tol):
            best = min(best, float(lp.c @ x))
    return best


def highs(lp) -> float:
    """Optimum value by scipy.optimize.linprog(method='highs')."""
    import scipy.sparse as sp
    from scipy.optimize import linprog
    K = sp.csr_matrix((lp.val, lp.col_idx.astype(np.int64), lp.row_ptr), shape=(lp.m, lp.n))
    G, A = K[: lp.m1], K[lp.m1:]
    bounds = list(zip([None if not np.isfinite(v) else v for v in lp.l],
                      [None if not np.isfinite(v) else v for v in lp.u]))
    res = linprog(lp.c, A_ub=-G if lp.m1 else None, b_ub=-lp.q[: lp.m1] if lp.m1 else None,
                  A_eq=A if lp.m2 else None, b_eq=lp.q[lp.m1:] if lp.m2 else None,
                  bounds=bounds, method="highs")
    assert res.status == 0, res.message
    return float(res.fun)
