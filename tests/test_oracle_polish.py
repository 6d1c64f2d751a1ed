"""Pins of the oracle's feasibility polishing (DESIGN.md §3
reading 36, acceptance #6 S:629).

Pinned against what polishing must achieve on the original data, recomputed
independently (`kkt_original`: fresh products with the unscaled K): the primal
residual of the returned x and the dual residual of the returned y reach
eps_feas_polish, the reduced costs are c - K'y, already-feasible points come
back at the first check, and an unfinished polish is flagged."""
import numpy as np
import pytest

import lpgen
import oracle

EPS_FP = 1e-6


def kkt(lp, r):
    return oracle.kkt_original(lp, r["x"], r["y"])


def polish_solve(lp, alg, **kw):
    return oracle.solve(lp, alg, feasibility_polishing=True, **kw)


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_acceptance_6_knapsack_and_grid(alg):
    """from eps 1e-3 solutions, polishing drives the primal residual <= 1e-6
    (relative form, reading 36) on every instance; the dual residual too; the
    objective change is reported (here: bounded by the main tolerance's scale)."""
    lps = [lpgen.random_small_lp(s, n=20, m1=3, m2=0) for s in range(25)]
    lp, C = lpgen.g_grid(batch=20, k=4)
    lps += [lp.with_costs(c=C[b]) for b in range(20)]
    worst = 0.0
    for lp in lps:
        r0 = oracle.solve(lp, alg, eps_abs=1e-3, eps_rel=1e-3)
        r = polish_solve(lp, alg, eps_abs=1e-3, eps_rel=1e-3)
        assert r0["status"] == r["status"] == oracle.OPTIMAL and r["polish"] == 1
        k = kkt(lp, r)
        nq, nc = np.linalg.norm(lp.q), np.linalg.norm(lp.c)
        assert k["pres"] <= (1 + 1e-9) * EPS_FP * (1 + nq), k["pres"]
        assert k["dres"] <= (1 + 1e-9) * EPS_FP * (1 + nc), k["dres"]
        # the result's fields are the polished pair's, on the original data
        assert r["primal_residual"] == pytest.approx(k["pres"], rel=1e-6, abs=1e-15)
        assert r["primal_objective"] == pytest.approx(float(lp.c @ r["x"]), rel=1e-12, abs=1e-14)
        worst = max(worst, abs(r["primal_objective"] - r0["primal_objective"]) / (1 + abs(r0["primal_objective"])))
        # iterations: the main solve's plus two polish solves of >= one check interval each
        assert r["iterations"] >= r0["iterations"] + 128
    assert worst <= 1e-2, worst


def test_dual_residual_polished_on_free_variables():
    """G-RAND has free and half-bounded columns, where dres > 0 before polishing."""
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    for alg in ("ra", "r2"):
        r0 = oracle.solve(lp, alg, eps_abs=1e-2, eps_rel=1e-2)
        r = polish_solve(lp, alg, eps_abs=1e-2, eps_rel=1e-2)
        k0, k = kkt(lp, r0), kkt(lp, r)
        nq, nc = np.linalg.norm(lp.q), np.linalg.norm(lp.c)
        assert k0["pres"] > EPS_FP * (1 + nq) and k0["dres"] > EPS_FP * (1 + nc)  # polishing has work to do
        assert k["pres"] <= (1 + 1e-9) * EPS_FP * (1 + nq)
        assert k["dres"] <= (1 + 1e-9) * EPS_FP * (1 + nc)
        assert np.allclose(r["lam"], lp.c - lp.dense_K().T @ r["y"], atol=1e-9)
        assert abs(r["primal_objective"] - lp.obj_star) <= 1e-2 * (1 + abs(lp.obj_star))


def test_already_feasible_point_is_returned_at_the_first_check():
    """a primal-feasible x* with y = 0 is a fixed point of the c = 0 iteration
    (x' = x, y' = [sigma (q - Kx)]^+ = 0), so the primal polish stops at its first
    check with x unchanged; likewise a dual-feasible y* (q = 0, x = proj(0) = 0)."""
    lp = lpgen.stack([1.0, 1.0], G=[[1.0, 1.0]], h=[1.0], l=[0.0, 0.0], u=[1.0, 1.0])
    # every x with x1 + x2 = 1 is optimal; the main solve stops at a feasible vertex or face point
    for alg in ("ra", "r2"):
        r0 = oracle.solve(lp, alg, eps_abs=1e-9, eps_rel=1e-9)
        k0 = kkt(lp, r0)
        r = polish_solve(lp, alg, eps_abs=1e-9, eps_rel=1e-9)
        assert k0["pres"] <= EPS_FP and r["polish"] == 1
        assert r["iterations"] == r0["iterations"] + 128          # one check interval per polish
        assert np.allclose(r["x"], r0["x"], rtol=0, atol=1e-6)


def test_zero_cost_problem():
    """with c = 0 the primal polish solves the main problem again (from x*)."""
    lp = lpgen.g_rand(50, 100, 10, seed=1).with_costs(c=np.zeros(100))
    r = polish_solve(lp, "ra", eps_abs=1e-3, eps_rel=1e-3)
    k = kkt(lp, r)
    assert r["status"] == oracle.OPTIMAL and r["polish"] == 1
    assert k["pres"] <= (1 + 1e-9) * EPS_FP * (1 + np.linalg.norm(lp.q))
    assert r["primal_objective"] == 0.0


def test_unfinished_polish_is_flagged():
    """a polish solve that reaches the iteration limit flags `polish = 2`; the
    status stays the main solve's OPTIMAL."""
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    r = oracle.solve(lp, "ra", eps_abs=1e-2, eps_rel=1e-2, iteration_limit=192,
                     feasibility_polishing=True, eps_feas_polish=1e-14)
    assert r["status"] == oracle.OPTIMAL and r["polish"] == 2


def test_no_polish_unless_optimal():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    r = oracle.solve(lp, "ra", eps_abs=1e-12, eps_rel=1e-12, iteration_limit=64, feasibility_polishing=True)
    r0 = oracle.solve(lp, "ra", eps_abs=1e-12, eps_rel=1e-12, iteration_limit=64)
    assert r["status"] == oracle.ITERATION_LIMIT and r["polish"] == 0
    assert np.array_equal(r["x"], r0["x"]) and r["iterations"] == 64
    inf = lpgen.g_infeasible("primal", 0)
    r = oracle.solve(inf, "ra", iteration_limit=10000, feasibility_polishing=True)
    assert r["status"] == oracle.PRIMAL_INFEASIBLE and r["polish"] == 0


def test_batch_polishing_equals_single():
    lp, C = lpgen.g_grid(batch=12, k=4)
    X, Y, res = oracle.solve_batch(lp, C, None, "r2", eps_abs=1e-3, eps_rel=1e-3, feasibility_polishing=True)
    for b in range(12):
        r = oracle.solve(lp.with_costs(c=C[b]), "r2", eps_abs=1e-3, eps_rel=1e-3, feasibility_polishing=True)
        assert np.array_equal(X[b], r["x"]) and np.array_equal(Y[b], r["y"])
        assert res[b]["iterations"] == r["iterations"] and res[b]["polish"] == r["polish"]
