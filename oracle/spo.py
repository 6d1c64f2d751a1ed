"""SPO+ loss and subgradient on top of the oracle's batch solve (TEST
INFRASTRUCTURE ONLY; see oracle/mpax_oracle.c's header for who may use it).

Plain numpy arithmetic of PAPER.md Eq. (spo+ loss) and Eq. (spo+
gradient), in the form of the listing P:198-215: the inner LPs
min_{x in S} (2c^ - c)'x are solved by `solve_batch`, obj = its primal objective,
  loss_b = -obj_b + 2 c^_b'x*(c_b) - c_b'x*(c_b),   grad_b = 2 x*(c_b) - 2 x_b."""
from __future__ import annotations

import numpy as np

from .oracle import solve_batch


def spo_plus(lp, C_pred, C_true, X_true, obj_true, algorithm="r2", X0=None, Y0=None, **kw):
    """Returns (loss[B], grad[B, n], X_inner, Y_inner, results)."""
    C_pred, C_true, X_true = (np.asarray(a, np.float64) for a in (C_pred, C_true, X_true))
    obj_true = np.asarray(obj_true, np.float64)
    C_in = 2.0 * C_pred - C_true
    X, Y, res = solve_batch(lp, C_in, None, algorithm, X0=X0, Y0=Y0, **kw)
    obj = np.array([r["primal_objective"] for r in res])
    loss = -obj + 2.0 * np.sum(C_pred * X_true, axis=1) - obj_true
    grad = 2.0 * (X_true - X)
    return loss, grad, X, Y, res
