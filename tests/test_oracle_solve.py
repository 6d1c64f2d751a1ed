"""End-to-end pins of the oracle's full solve (contract steps 0-6) against the
plain definition of the LP optimum, Eq. (1): brute-force
vertex enumeration, dynamic programming on the totally unimodular grid flow
LP, the constructed optimum of G-RAND (strong duality), HiGHS,
and the optimality conditions themselves.  CPU only.

Iteration / attempt / restart COUNTS are parity unpinned externally (the
paper's counts need its datasets); tests here only check they are sane."""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle
from tests import truth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
ALGS = ["ra", "r2"]


@pytest.mark.parametrize("alg", ALGS)
def test_tiny_spec_s435(alg):
    g = GOLD["solve_tiny"]
    r = oracle.solve(lpgen.tiny_spec(), alg, eps_abs=g["eps"], eps_rel=g["eps"])
    assert r["status"] == oracle.OPTIMAL
    assert abs(r["primal_objective"] - g["objective"]) <= g["tol"]
    assert np.allclose(r["x"], g["x"], atol=1e-6)


@pytest.mark.parametrize("alg", ALGS)
def test_warm_start_at_optimum_s436(alg):
    g = GOLD["warm_start_optimum"]
    r = oracle.solve(lpgen.tiny_spec(), alg, x0=g["x0"], y0=g["y0"])
    assert r["status"] == oracle.OPTIMAL and r["iterations"] == g["first_check"]
    assert np.allclose(r["x"], g["x0"], rtol=0, atol=1e-15)   # x0 / Dc * Dc round trip


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("seed", range(8))
def test_vertex_enumeration_s624(alg, seed):
    lp = lpgen.random_small_lp(seed, n=4, m1=2, m2=1)
    best = truth.vertex_enumeration(lp)
    r = oracle.solve(lp, alg, eps_abs=1e-8, eps_rel=1e-8, iteration_limit=400000)
    assert r["status"] == oracle.OPTIMAL
    assert abs(r["primal_objective"] - best) <= 1e-6 * (1 + abs(best))


@pytest.mark.parametrize("alg", ALGS)
def test_grid_dp(alg):
    lp, C = lpgen.g_grid(batch=8)
    X, Y, res = oracle.solve_batch(lp, C, None, alg, eps_abs=1e-8, eps_rel=1e-8, iteration_limit=400000)
    for b in range(8):
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert res[b]["status"] == oracle.OPTIMAL
        assert abs(res[b]["primal_objective"] - dp) <= 1e-6 * (1 + dp)
    X4, _, res4 = oracle.solve_batch(lp, C, None, alg)             # 1e-4 sanity (SURVEY c.4)
    for b in range(8):
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert res4[b]["status"] == oracle.OPTIMAL
        assert abs(res4[b]["primal_objective"] - dp) <= 1e-3 * (1 + dp)


@pytest.mark.parametrize("alg", ALGS)
def test_grand_known_optimum(alg):
    lp = lpgen.g_rand(50, 100, 10, seed=1)                           # C1
    r = oracle.solve(lp, alg, eps_abs=1e-8, eps_rel=1e-8, iteration_limit=400000)
    assert r["status"] == oracle.OPTIMAL
    assert abs(r["primal_objective"] - lp.obj_star) <= 1e-6 * (1 + abs(lp.obj_star))
    r4 = oracle.solve(lp, alg)
    assert r4["status"] == oracle.OPTIMAL and r4["rel_kkt"] <= 1e-4
    assert abs(r4["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))


@pytest.mark.parametrize("alg", ALGS)
def test_highs(alg):
    lp = lpgen.g_rand(300, 600, 8, seed=21)
    ref = truth.highs(lp)
    assert abs(ref - lp.obj_star) <= 1e-7 * (1 + abs(ref))      # the generator's optimum, independently
    r = oracle.solve(lp, alg, eps_abs=1e-8, eps_rel=1e-8, iteration_limit=400000)
    assert r["status"] == oracle.OPTIMAL
    assert abs(r["primal_objective"] - ref) <= 1e-6 * (1 + abs(ref))


@pytest.mark.parametrize("alg", ALGS)
def test_optimality_invariants(alg):
    """Self-certification and complementary slackness / strong duality
     at the returned solution."""
    lp = lpgen.g_rand(80, 160, 8, seed=9)
    eps = 1e-6
    r = oracle.solve(lp, alg, eps_abs=eps, eps_rel=eps)
    assert r["status"] == oracle.OPTIMAL
    x, y = r["x"], r["y"]
    assert np.all(x >= lp.l) and np.all(x <= lp.u) and np.all(y[: lp.m1] >= 0)
    k = oracle.kkt_original(lp, x, y)
    nq, nc = np.linalg.norm(lp.q), np.linalg.norm(lp.c)
    slack = 1 + 1e-9
    assert k["pres"] <= slack * (eps + eps * nq)
    assert k["dres"] <= slack * (eps + eps * nc)
    assert k["gap"] <= slack * (eps + eps * (abs(k["pobj"]) + abs(k["dobj"])))
    Kx, KTy = oracle.spmv_pair(lp, x=x, w=y)
    lam = lp.c - KTy
    assert np.allclose(lam, r["lam"], rtol=1e-10, atol=1e-10)
    scale = 1 + np.abs(lp.obj_star)
    assert abs(np.sum(y[: lp.m1] * (Kx[: lp.m1] - lp.q[: lp.m1]))) <= 1e3 * eps * scale
    fl = np.isfinite(lp.l)
    assert abs(np.sum(np.maximum(lam, 0)[fl] * (x[fl] - lp.l[fl]))) <= 1e3 * eps * scale


def test_batch_equals_map_and_identical_instances_s455_464():
    lp, C = lpgen.g_grid(batch=6)
    C[3] = C[1]
    X, Y, res = oracle.solve_batch(lp, C, None, "r2")
    for b in range(6):
        r = oracle.solve(lp.with_costs(c=C[b]), "r2")
        assert np.array_equal(r["x"], X[b]) and np.array_equal(r["y"], Y[b])
        assert r["iterations"] == res[b]["iterations"]
    assert np.array_equal(X[3], X[1]) and np.array_equal(Y[3], Y[1])


def test_thread_count_independence_and_determinism():
    lp = lpgen.g_rand(2000, 4000, 10, seed=4)
    t0 = oracle.num_threads()
    oracle.set_threads(1)
    a = oracle.solve(lp, "ra", iteration_limit=128)
    oracle.set_threads(max(t0, 4))
    b = oracle.solve(lp, "ra", iteration_limit=128)
    c = oracle.solve(lp, "ra", iteration_limit=128)
    oracle.set_threads(t0)
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(b["x"], c["x"])
    assert a["attempts"] == b["attempts"] == c["attempts"]


@pytest.mark.parametrize("alg", ALGS)
def test_iteration_limit_and_degenerate(alg):
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    r = oracle.solve(lp, alg, eps_abs=1e-12, eps_rel=1e-12, iteration_limit=100)
    assert r["status"] == oracle.ITERATION_LIMIT and r["iterations"] == 100
    assert r["attempts"] >= 100
    # no constraints (m = 0): min c'x over a box -> each x_j at its cheap bound
    lp0 = lpgen.stack([1.0, -2.0, 0.5], l=[-1, -1, 0], u=[1, 3, 2])
    r = oracle.solve(lp0, alg, eps_abs=1e-9, eps_rel=1e-9)
    assert r["status"] == oracle.OPTIMAL and np.allclose(r["x"], [-1, 3, 0], atol=1e-8)
    # K with an all-zero row and column
    lpz = lpgen.stack([1.0, 1.0], G=[[1.0, 0.0], [0.0, 0.0]], h=[1.0, -1.0], l=[0, 0], u=[5, 5])
    r = oracle.solve(lpz, alg, eps_abs=1e-9, eps_rel=1e-9)
    assert r["status"] == oracle.OPTIMAL and abs(r["primal_objective"] - 1.0) <= 1e-7


@pytest.mark.parametrize("alg", ALGS)
def test_constant_step_variant(alg):
    """Constant step eta = 0.998 / sigma_max(K~): no line search,
    so every attempt is accepted; same optima (plain definitions as above)."""
    r = oracle.solve(lpgen.tiny_spec(), alg, eps_abs=1e-8, eps_rel=1e-8, step_rule=1)
    assert r["status"] == oracle.OPTIMAL and abs(r["primal_objective"] - 1.0) <= 1e-6
    assert r["attempts"] == r["iterations"]
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    r = oracle.solve(lp, alg, eps_abs=1e-8, eps_rel=1e-8, iteration_limit=400000, step_rule=1)
    assert r["status"] == oracle.OPTIMAL and r["attempts"] == r["iterations"]
    assert abs(r["primal_objective"] - lp.obj_star) <= 1e-6 * (1 + abs(lp.obj_star))
    lpg, C = lpgen.g_grid(batch=16)
    _, _, res = oracle.solve_batch(lpg, C, None, alg, step_rule=1)
    for b in range(16):
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert res[b]["status"] == oracle.OPTIMAL and abs(res[b]["primal_objective"] - dp) <= 1e-3 * (1 + dp)
        assert res[b]["attempts"] == res[b]["iterations"]


# ---- partial reflection (reading 38) ----

def test_partial_reflection_step_pins():
    rng = np.random.default_rng(5)
    z, w, z0 = rng.normal(size=(3, 17))
    for k in (0, 3, 40):
        # rho = 1 is the full reflection of P:64, the same operations bit for bit
        assert np.array_equal(oracle.halpern_rho(k, z, w, z0, 1.0), oracle.halpern(k, z, w, z0))
        # a fixed point of the PDHG map (w = z) anchored at itself stays put for every rho
        for rho in (0.0, 0.3, 1.0):
            assert np.allclose(oracle.halpern_rho(k, z, z, z, rho), z, rtol=1e-15, atol=1e-15)
    # rho = 0, k = 0: plain Halpern on PDHG, (w + z0) / 2 (a = b = 1/2)
    assert np.allclose(oracle.halpern_rho(0, z, w, z0, 0.0), 0.5 * w + 0.5 * z0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("rho", [0.0, 0.5, 0.9])
def test_partial_reflection_solves(rho):
    """Partial reflection reaches the same optima (constructed G-RAND optimum, grid DP);
    rho = 1 is bitwise the default; rho outside [0, 1] is rejected."""
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    r = oracle.solve(lp, "r2", reflection=rho)
    assert r["status"] == oracle.OPTIMAL
    assert abs(r["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))
    grid, C = lpgen.g_grid(batch=32)
    _, _, res = oracle.solve_batch(grid, C, None, "r2", reflection=rho)
    for b in range(32):
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert res[b]["status"] == oracle.OPTIMAL and abs(res[b]["primal_objective"] - dp) <= 1e-3 * (1 + dp)
    a, b_ = oracle.solve(lp, "r2", reflection=1.0), oracle.solve(lp, "r2")
    assert np.array_equal(a["x"], b_["x"]) and a["attempts"] == b_["attempts"]
    with pytest.raises(ValueError):
        oracle.solve(lp, "r2", reflection=1.5)


def _restart_kinds(chk):
    """Classify each logged restart by the first criterion of reading 12 it meets."""
    kinds, last_k = [], 0
    for k, metric, ref, last, rs, ps in chk[:, :6]:
        if rs == 1:
            kinds.append("artificial" if k - last_k >= 0.36 * k else "sufficient" if metric <= 0.2 * ref else "necessary")
            last_k = k
    return kinds


def test_r2_adaptive_tail_mechanism():
    """DESIGN.md reading 31: why adaptive-step r2HPDHG has a heavy tail on C2 (the oracle's
    slowest instance of the 1024-LP batch, 6976 iterations vs a median of 192).  After a
    sufficient restart at an excellent point the epoch's reference r_P(first step) is tiny, the
    fixed-point residual then GROWS by >100x under the adaptive step (the line search bounds
    <dy, K dx> only, which does not keep the reflected Halpern map nonexpansive), so neither the
    sufficient nor the necessary test can fire and the epoch ends only at the artificial
    k_in >= 0.36 k: epochs grow geometrically (x1.56).  With the constant step (reading 34) the
    same LP takes <= 576 iterations."""
    lp, C = lpgen.g_grid(batch=1024, seed=2)
    lpb = lp.with_costs(c=C[764])
    r = oracle.solve(lpb, "r2", log_capacity=1 << 16)
    assert r["status"] == oracle.OPTIMAL and r["iterations"] >= 4000
    chk = r["chk_log"]
    kinds = _restart_kinds(chk)
    assert "necessary" not in kinds and kinds.count("artificial") >= 6
    # the long epochs: each starts right after a sufficient restart and ends artificially
    ks = [int(k) for k, rs in zip(chk[:, 0], chk[:, 4]) if rs == 1]
    long_epochs = [(a, b) for a, b, t in zip(ks, ks[1:], kinds[1:]) if b - a > 256]
    assert len(long_epochs) >= 3 and all(kinds[ks.index(b)] == "artificial" for _, b in long_epochs)
    assert all(kinds[ks.index(a)] == "sufficient" for a, _ in long_epochs)
    ratio = chk[:, 1] / chk[:, 2]
    assert ratio.max() > 100.0                      # the residual grows far above the epoch's reference
    lens = [b - a for a, b in long_epochs]
    assert all(l2 > 1.4 * l1 for l1, l2 in zip(lens, lens[1:]))   # geometric epoch growth
    rc = oracle.solve(lpb, "r2", step_rule="constant")
    assert rc["status"] == oracle.OPTIMAL and rc["iterations"] <= 576
