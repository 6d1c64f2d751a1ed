"""Pins of the oracle's infeasibility detection (DESIGN.md §3
reading 35, acceptance #7 S:630; tolerances P:530-531).

The certificate test is pinned on hand-checked Farkas certificates (SPEC
S:425-426 and bound-term examples worked below); the full solves are pinned
against an independent classifier (scipy's HiGHS, a library LP solver) on
planted infeasible instances, and every returned ray is re-checked against
the Farkas alternative written with the support function of the box."""
import numpy as np
import pytest

import lpgen
import oracle

INF = np.inf
PI, DI = oracle.PRIMAL_INFEASIBLE, oracle.DUAL_INFEASIBLE


def spec_primal_infeasible():
    """x >= 1 and -x >= 0 (i.e. x <= 0), x free."""
    return lpgen.stack([0.0], G=[[1.0], [-1.0]], h=[1.0, 0.0], l=[-INF], u=[INF])


def spec_dual_infeasible():
    """min -x, x >= 0, no constraints."""
    return lpgen.stack([-1.0], l=[0.0], u=[INF])


# ------------------------------------------------------- the certificate test

def test_spec_farkas_dual_ray():
    """d_y = (1, 1)/sqrt2 certifies x >= 1, x <= 0: q'd_y = 1/sqrt2 > 0, K'd_y = 0."""
    c = oracle.certificate_test(spec_primal_infeasible(), [0.0], np.array([1.0, 1.0]) / np.sqrt(2))
    assert c["primal_infeasible"] == 1 and c["dual_infeasible"] == 0
    assert c["dual_ray_objective"] == pytest.approx(1 / np.sqrt(2), rel=1e-15)
    assert c["dual_ray_violation"] == 0.0
    # the unnormalised ray gives the same verdict (the test scales to unit norm)
    c2 = oracle.certificate_test(spec_primal_infeasible(), [0.0], [3.0, 3.0])
    assert c2["primal_infeasible"] == 1 and c2["dual_ray_objective"] == pytest.approx(1 / np.sqrt(2), rel=1e-15)
    # an unbalanced ray leaves K'd_y = 1 on a free column: not a certificate
    c3 = oracle.certificate_test(spec_primal_infeasible(), [0.0], [2.0, 1.0])
    assert c3["primal_infeasible"] == 0 and c3["dual_ray_violation"] == pytest.approx(1 / np.sqrt(5), rel=1e-15)
    # a negative multiplier on a ">=" row is a violation
    c4 = oracle.certificate_test(spec_primal_infeasible(), [0.0], [-1.0, -1.0])
    assert c4["primal_infeasible"] == 0


def test_spec_unbounded_primal_ray():
    """d_x = 1 certifies min -x, x >= 0: c'd_x = -1 < 0."""
    c = oracle.certificate_test(spec_dual_infeasible(), [1.0], np.zeros(0))
    assert c["dual_infeasible"] == 1 and c["primal_infeasible"] == 0
    assert c["primal_ray_objective"] == -1.0 and c["primal_ray_violation"] == 0.0
    # the opposite direction leaves the finite lower bound: violation 1, no certificate
    c2 = oracle.certificate_test(spec_dual_infeasible(), [-1.0], np.zeros(0))
    assert c2["dual_infeasible"] == 0 and c2["primal_ray_violation"] == 1.0


def test_bound_terms_of_the_dual_ray():
    """x >= 2 with 0 <= x <= 1 is infeasible through the box: d_y = 1 gives
    lambda = -K'd_y = -1, so the dual-ray objective is q'd_y - u lambda^- = 2 - 1 = 1."""
    lp = lpgen.stack([0.0], G=[[1.0]], h=[2.0], l=[0.0], u=[1.0])
    c = oracle.certificate_test(lp, [0.0], [1.0])
    assert c["primal_infeasible"] == 1 and c["dual_ray_objective"] == 1.0
    # with u = 2 the same ray has objective 0: x = 2 is feasible, no certificate
    lp2 = lpgen.stack([0.0], G=[[1.0]], h=[2.0], l=[0.0], u=[2.0])
    assert oracle.certificate_test(lp2, [0.0], [1.0])["primal_infeasible"] == 0
    # lower-bound term: -x >= 1 with -1 <= x <= 5 is infeasible: lambda = +1, objective 1 + l*1 = 0 -> not
    # a certificate at l = -1, a certificate at l = -0.5 (objective 0.5)
    lp3 = lpgen.stack([0.0], G=[[-1.0]], h=[1.0], l=[-1.0], u=[5.0])
    assert oracle.certificate_test(lp3, [0.0], [1.0])["primal_infeasible"] == 0
    lp4 = lpgen.stack([0.0], G=[[-1.0]], h=[1.0], l=[-0.5], u=[5.0])
    c4 = oracle.certificate_test(lp4, [0.0], [1.0])
    assert c4["primal_infeasible"] == 1 and c4["dual_ray_objective"] == 0.5


def test_primal_ray_row_terms():
    """x1 - x2 = 0 and x1 + x2 >= 0 with x >= 0 free above, c = (-1, 0): d_x = (1, 1)
    is a recession direction (A d = 0, G d = 2 >= 0) with c'd < 0; (1, 0) breaks the
    equality row and (1, -1) the ">=" row and the bound."""
    lp = lpgen.stack([-1.0, 0.0], G=[[1.0, 1.0]], h=[0.0], A=[[1.0, -1.0]], b=[0.0], l=[0.0, 0.0], u=[INF, INF])
    c = oracle.certificate_test(lp, [1.0, 1.0], [0.0, 0.0])
    assert c["dual_infeasible"] == 1 and c["primal_ray_objective"] == pytest.approx(-1 / np.sqrt(2), rel=1e-15)
    c2 = oracle.certificate_test(lp, [1.0, 0.0], [0.0, 0.0])
    assert c2["dual_infeasible"] == 0 and c2["primal_ray_violation"] == 1.0
    c3 = oracle.certificate_test(lp, [-1.0, -2.0], [0.0, 0.0])
    assert c3["dual_infeasible"] == 0


def test_negative_tolerance_disables_the_test():
    c = oracle.certificate_test(spec_primal_infeasible(), [0.0], [1.0, 1.0], eps_primal_infeasible=-1.0)
    assert c["primal_infeasible"] == 0


# ------------------------------------------------------------- full solves

def scipy_status(lp):
    """HiGHS classification: 0 optimal, 2 infeasible, 3 unbounded."""
    from scipy.optimize import linprog
    K = lp.dense_K()
    G, A = K[: lp.m1], K[lp.m1:]
    bounds = [(None if not np.isfinite(a) else a, None if not np.isfinite(b) else b) for a, b in zip(lp.l, lp.u)]
    r = linprog(lp.c, A_ub=-G if lp.m1 else None, b_ub=-lp.q[: lp.m1] if lp.m1 else None,
                A_eq=A if lp.m2 else None, b_eq=lp.q[lp.m1:] if lp.m2 else None, bounds=bounds, method="highs")
    return r.status


def farkas_primal_ok(lp, y, tol=1e-7):
    """y (unit) proves {Kx >=/= q, l <= x <= u} empty: y_G >= 0 and
    q'y > sup_{x in box} (K'y)'x (support function of the box), within tol."""
    K = lp.dense_K()
    r = K.T @ y
    if np.any(y[: lp.m1] < -tol):
        return False
    if np.any((r > tol) & ~np.isfinite(lp.u)) or np.any((r < -tol) & ~np.isfinite(lp.l)):
        return False
    sup = np.sum(np.where(r > 0, r * np.where(np.isfinite(lp.u), lp.u, 0.0),
                          r * np.where(np.isfinite(lp.l), lp.l, 0.0)))
    return lp.q @ y - sup > tol


def farkas_dual_ok(lp, x, tol=1e-7):
    """x (unit) is a recession direction with c'x < 0."""
    K = lp.dense_K()
    Kx = K @ x
    return (lp.c @ x < -tol and np.all(Kx[: lp.m1] >= -tol) and np.all(np.abs(Kx[lp.m1:]) <= tol)
            and np.all(x[np.isfinite(lp.u)] <= tol) and np.all(x[np.isfinite(lp.l)] >= -tol))


CASES = [(alg, rule) for alg in ("ra", "r2") for rule in (0, 1)]


@pytest.mark.parametrize("alg,rule", CASES)
@pytest.mark.parametrize("kind", ["primal", "dual"])
def test_planted_infeasible_instances(alg, rule, kind):
    """20 planted instances per kind, classified by HiGHS; the oracle must return
    the matching status within 10,000 iterations, with a ray that passes
    the Farkas check -- except adaptive-step r2HPDHG on primal-infeasible LPs, whose
    iterates grow geometrically (reading 35): there it must never return
    a wrong classification."""
    want = PI if kind == "primal" else DI
    hits = 0
    for s in range(20):
        lp = lpgen.g_infeasible(kind, s)
        assert scipy_status(lp) == (2 if kind == "primal" else 3)
        r = oracle.solve(lp, alg, iteration_limit=10000, step_rule=rule)
        assert r["status"] in (want, oracle.ITERATION_LIMIT, oracle.NUMERICAL_ERROR), r["status"]
        if r["status"] == want:
            hits += 1
            assert r["iterations"] % 64 == 0
            if kind == "primal":
                assert abs(np.linalg.norm(r["y"]) - 1) <= 1e-12 and farkas_primal_ok(lp, r["y"])
            else:
                assert abs(np.linalg.norm(r["x"]) - 1) <= 1e-12 and farkas_dual_ok(lp, r["x"])
    assert hits >= (10 if (alg, rule, kind) == ("r2", 0, "primal") else 20), hits


@pytest.mark.parametrize("alg,rule", CASES)
def test_spec_examples(alg, rule):
    r = oracle.solve(spec_dual_infeasible(), alg, iteration_limit=10000, step_rule=rule)
    assert r["status"] == DI and r["x"][0] == 1.0
    r = oracle.solve(spec_primal_infeasible(), alg, iteration_limit=10000, step_rule=rule)
    if (alg, rule) == ("r2", 0):
        assert r["status"] in (oracle.ITERATION_LIMIT, oracle.NUMERICAL_ERROR)
    else:
        assert r["status"] == PI
        assert np.allclose(r["y"], [1 / np.sqrt(2)] * 2, rtol=1e-7)


def test_feasible_instances_are_not_flagged():
    """No false certificate on feasible LPs (HiGHS: optimal) with either rule."""
    lps = [lpgen.random_small_lp(s, n=10, m1=5, m2=3) for s in range(15)]
    for lp in lps:
        assert scipy_status(lp) == 0
        for alg, rule in CASES:
            assert oracle.solve(lp, alg, step_rule=rule)["status"] == oracle.OPTIMAL


def test_batch_mixes_statuses():
    """A batch sharing K where some cost vectors make the LP unbounded."""
    lp = lpgen.g_infeasible("dual", 3)
    j = int(np.nonzero(~np.isfinite(lp.u))[0][0])
    C = np.tile(lp.c, (6, 1))
    C[::2, j] = np.abs(C[::2, j]) + 1.0          # even rows: c_j > 0, the LP is bounded
    _, _, res = oracle.solve_batch(lp, C, None, "ra", iteration_limit=20000)
    for b in range(6):
        want = oracle.OPTIMAL if b % 2 == 0 else DI
        assert scipy_status(lp.with_costs(c=C[b])) == (0 if b % 2 == 0 else 3)
        assert res[b]["status"] == want, (b, res[b]["status"])
