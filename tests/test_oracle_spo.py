"""Pins of the oracle's SPO+ loss / subgradient (PAPER.md
Eq. (spo+ loss) P:76-78, Eq. (spo+ gradient) P:80-82, listing P:198-215; SPEC
S:511-536, acceptance #8 S:631).

Pinned by the SPEC's hand-evaluated examples, by the loss's algebra at c^ = c,
by the SPO+ properties (nonnegativity for exact x*(c), subgradient bounded by
the box), by exact inner solutions from a library LP solver (HiGHS), and by
central finite differences of the loss."""
import numpy as np
import pytest
from scipy.optimize import linprog

import lpgen
import oracle
from oracle.spo import spo_plus

TIGHT = dict(eps_abs=1e-10, eps_rel=1e-10)


def highs(lp, c):
    """Exact vertex solution of min c'x over S (K, q, l, u of lp) and its value."""
    K = lp.dense_K()
    G, A = K[: lp.m1], K[lp.m1:]
    bounds = [(None if not np.isfinite(a) else a, None if not np.isfinite(b) else b) for a, b in zip(lp.l, lp.u)]
    r = linprog(c, A_ub=-G if lp.m1 else None, b_ub=-lp.q[: lp.m1] if lp.m1 else None,
                A_eq=A if lp.m2 else None, b_eq=lp.q[lp.m1:] if lp.m2 else None, bounds=bounds,
                method="highs-ds")
    assert r.status == 0
    return r.x, r.fun


def test_spec_interval_example():
    """S = [0, 1], c = -1, c^ = +1: 2c^ - c = 3, inner min 0 at x = 0,
    loss = 0 + 2*1*1 - (-1)*1 = 3, subgradient 2*1 - 2*0 = 2."""
    lp = lpgen.stack([0.0], l=[0.0], u=[1.0])
    loss, grad, X, _, res = spo_plus(lp, [[1.0]], [[-1.0]], [[1.0]], [-1.0], "ra", **TIGHT)
    assert res[0]["status"] == oracle.OPTIMAL
    assert loss[0] == pytest.approx(3.0, abs=1e-9) and grad[0, 0] == pytest.approx(2.0, abs=1e-9)


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_perfect_prediction_gives_zero(alg):
    """c^ = c -> loss = -c'x*(c) + 2c'x*(c) - c'x*(c) = 0 and, with a unique
    optimum, gradient 0 (the inner solution is x*(c))."""
    k = 6
    lp = lpgen.warcraft_lp(k)
    C = lpgen.warcraft_costs(k, 4, seed=3, noise=0.3)        # generic costs: unique shortest paths
    Xt = np.stack([highs(lp, C[b])[0] for b in range(4)])
    ot = np.sum(C * Xt, axis=1)
    loss, grad, _, _, res = spo_plus(lp, C, C, Xt, ot, alg, **TIGHT)
    assert np.all(np.abs(loss) <= 1e-7 * (1 + np.abs(ot)))
    assert np.abs(grad).max() <= 1e-6


def test_batch_of_identical_members():
    lp = lpgen.knapsack_lp(12, 2, seed=1, dense=False)
    V = lpgen.knapsack_values(12, 1, seed=2)
    Xt, ot = highs(lp, V[0])
    P = V * 0.7
    l1, g1, *_ = spo_plus(lp, P, V, Xt[None], [ot], "ra", **TIGHT)
    l2, g2, *_ = spo_plus(lp, np.repeat(P, 2, 0), np.repeat(V, 2, 0), np.repeat(Xt[None], 2, 0), [ot, ot], "ra",
                          **TIGHT)
    assert np.array_equal(l2, np.repeat(l1, 2)) and np.array_equal(g2, np.repeat(g1, 2, 0))


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_nonnegative_and_bounded_with_exact_true_solutions(alg):
    """loss >= 0 when x*(c) is truly optimal; for S inside [0, 1]^n every
    subgradient entry lies in [-2, 2]; and with HiGHS's exact inner solutions the loss and
    gradient equal the oracle's up to the inner tolerance (acceptance #8)."""
    rng = np.random.default_rng(7)
    for s in range(10):
        lp = lpgen.knapsack_lp(8, 2, seed=s, dense=False)
        V = lpgen.knapsack_values(8, 1, seed=100 + s, noise=0.5)
        Xt, ot = highs(lp, V[0])
        P = V * rng.uniform(0.2, 1.8, size=V.shape) + rng.normal(scale=0.1, size=V.shape)
        loss, grad, X, _, res = spo_plus(lp, P, V, Xt[None], [ot], alg, **TIGHT)
        assert res[0]["status"] == oracle.OPTIMAL
        assert loss[0] >= -1e-8 and np.all(np.abs(grad) <= 2 + 1e-9)
        xe, fe = highs(lp, 2 * P[0] - V[0])
        loss_exact = -fe + 2 * P[0] @ Xt - ot
        assert loss[0] == pytest.approx(loss_exact, abs=1e-7 * (1 + abs(loss_exact)))
        if np.abs(X[0] - xe).max() <= 1e-6:             # unique inner optimum: the same subgradient
            assert np.abs(grad[0] - 2 * (Xt - xe)).max() <= 1e-5


def test_finite_differences():
    """at generic points the subgradient matches central differences of the loss
    (h = 1e-5) to 1e-4, skipping members whose inner optimum changes across the step."""
    checked = 0
    for s in range(10):
        lp = lpgen.knapsack_lp(8, 2, seed=s, dense=False)
        V = lpgen.knapsack_values(8, 1, seed=200 + s, noise=0.5)
        Xt, ot = highs(lp, V[0])
        P = V * np.random.default_rng(s).uniform(0.5, 1.5, size=V.shape)
        _, grad, X, _, _ = spo_plus(lp, P, V, Xt[None], [ot], "ra", **TIGHT)
        h = 1e-5
        for j in range(lp.n):
            E = np.zeros_like(P)
            E[0, j] = h
            lp_, _, Xp, _, _ = spo_plus(lp, P + E, V, Xt[None], [ot], "ra", **TIGHT)
            lm_, _, Xm, _, _ = spo_plus(lp, P - E, V, Xt[None], [ot], "ra", **TIGHT)
            if np.abs(Xp - Xm).max() > 1e-6 or np.abs(Xp - X).max() > 1e-6:
                continue                                   # basis change across the perturbation
            fd = (lp_[0] - lm_[0]) / (2 * h)
            assert abs(fd - grad[0, j]) <= 1e-4, (s, j, fd, grad[0, j])
            checked += 1
    assert checked >= 40


def test_acceptance_9_training_loop_on_the_oracle():
    """S:632 on the oracle: plain gradient descent on the mean SPO+ loss of a linear predictor
    (50 knapsack samples, N = 20, d = 3, noiseless polynomial values, eps 1e-4) cuts the training
    loss by >= 50% and reaches a normalized test regret < 5% within 30 epochs (the GPU layer is
    held to the same bar in test_gpu_spo_training.py)."""
    N, D, P = 20, 3, 5
    lp = lpgen.knapsack_lp(N, D, seed=7, capacity=30.0, dense=False)
    B = (np.random.default_rng(8).uniform(size=(N, P)) < 0.5).astype(np.float64)

    def dataset(n, seed):
        rng = np.random.default_rng(seed)
        F = rng.normal(size=(n, P))
        return F, -(((F @ B.T) / np.sqrt(P) + 3.0) ** 4 + 1.0) / 3.5 ** 4

    Ftr, Ctr = dataset(50, 9)
    Fte, Cte = dataset(50, 10)
    kw = dict(step_rule=1, eps_abs=1e-4, eps_rel=1e-4)
    Xtr, _, _ = oracle.solve_batch(lp, Ctr, None, "r2", **kw)
    Xte, _, _ = oracle.solve_batch(lp, Cte, None, "r2", **kw)
    otr, ote = (Ctr * Xtr).sum(1), (Cte * Xte).sum(1)
    W, b = 0.1 * np.random.default_rng(0).normal(size=(N, P)), np.zeros(N)
    losses = []
    for _ in range(30):
        loss, grad, *_ = spo_plus(lp, Ftr @ W.T + b, Ctr, Xtr, otr, "r2", **kw)
        losses.append(loss.mean())
        g = grad / 50
        W -= 0.5 * (g.T @ Ftr)
        b -= 0.5 * g.sum(0)
    Xh, _, _ = oracle.solve_batch(lp, Fte @ W.T + b, None, "r2", **kw)
    regret = ((Cte * Xh).sum(1) - ote).sum() / np.abs(ote).sum()
    assert losses[-1] <= 0.5 * losses[0] and regret < 0.05, (losses[0], losses[-1], regret)
