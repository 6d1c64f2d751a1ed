"""GPU parity of the constant-step variant (DESIGN.md §3
reading 34) against the oracle's step_rule = 1: eta = 0.998 / sigma_max(K~)
from 200 power iterations with the same deterministic start vector, every
attempt accepted.  Every solver path (tiny register kernel, generic
per-instance kernel, persistent grid kernel, DMMA cluster kernel, row-sharded
engine) is held to the same bars as the adaptive rule (test_gpu_parity.py)."""
import dataclasses

import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from tests.test_gpu_parity import batch_drift, gpu_solve, oracle_stability, rel, small_lps  # noqa: E402

ALGS = ["ra", "r2"]
CONST = dict(step_rule="constant")


def oracle_eta(lp):
    """0.998 / sigma_max(K~) with K~ the oracle's scaled matrix (step 1)."""
    kt = dataclasses.replace(lp, val=oracle.scaled_problem(lp)["Kv"].copy())
    s = oracle.spectral_norm(kt, 200)
    return 0.998 / s if s > 0 else 1.0


# the single-CTA power kernel (small) and the multi-kernel one (m + n > 16384)
@pytest.mark.parametrize("name,lp", list(small_lps()) + [("big", lpgen.g_rand(12000, 20000, 8, seed=4))])
def test_constant_step_size_matches_oracle(name, lp):
    rg = gpu_solve(lp, "r2", iteration_limit=1, eps_abs=0.0, eps_rel=0.0, **CONST)
    assert rg["attempts"] == 1 and rg["iterations"] == 1
    # power iteration in a different summation order: agreement to a few ulps of
    # the converged quotient (the start vector and iteration count are identical)
    assert abs(rg["eta"] - oracle_eta(lp)) <= 1e-12 * oracle_eta(lp), (rg["eta"], oracle_eta(lp))


def test_constant_step_zero_matrix_and_no_rows():
    lpz = lpgen.stack([1.0, 1.0], G=[[0.0, 0.0]], h=[-1.0], l=[0, 0], u=[5, 5])
    rg = gpu_solve(lpz, "r2", iteration_limit=3, eps_abs=0.0, eps_rel=0.0, **CONST)
    assert rg["eta"] == 1.0 and rg["attempts"] == 3
    lp0 = lpgen.stack([1.0, -2.0, 0.5], l=[-1, -1, 0], u=[1, 3, 2])
    rg = gpu_solve(lp0, "ra", eps_abs=1e-9, eps_rel=1e-9, **CONST)
    assert rg["status"] == mp.LP_OPTIMAL and np.allclose(rg["x"], [-1, 3, 0], atol=1e-8)


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 64, 256])
@pytest.mark.parametrize("name,lp", list(small_lps()))
def test_constant_step_fixed_K(alg, K, name, lp):
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=K, **CONST)
    ro, stable, drift = oracle_stability(lp, alg, **kw)
    rg = gpu_solve(lp, alg, **kw)
    # no line search: attempts == accepted steps (fewer than K only when exactly optimal)
    assert rg["attempts"] == rg["iterations"] <= K
    if not stable:
        pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rel(rg["x"], ro["x"]) <= tol
    if lp.m:
        assert rel(rg["y"], ro["y"]) <= tol


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("name,lp", list(small_lps()))
def test_constant_step_full_solve(alg, name, lp):
    ro, stable, _ = oracle_stability(lp, alg, **CONST)
    rg = gpu_solve(lp, alg, **CONST)
    assert rg["status"] == mp.LP_OPTIMAL and ro["status"] == oracle.OPTIMAL
    assert rg["attempts"] == rg["iterations"]
    if stable:
        assert rg["iterations"] == ro["iterations"] and rg["restarts"] == ro["restarts"]
    assert rg["rel_kkt"] <= 1e-4
    k = oracle.kkt_original(lp, rg["x"], rg["y"])
    assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.q))
    assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.c))
    if lp.obj_star is not None:
        assert abs(rg["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))


@pytest.mark.parametrize("alg", ALGS)
def test_constant_step_c2_batch(alg):
    """C2 (1024 grid shortest-path LPs) with the constant step: fixed K = 64 parity
    on every count-stable instance, then full solves at the DP optimum."""
    lp, C = lpgen.g_grid(batch=1024)
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=64, **CONST)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    res = bs.solve(algorithm=alg, **kw)
    X, Y = bs.solutions()
    Xo, Yo, ro = oracle.solve_batch(lp, C, None, alg, **kw)
    stable, dx, _ = batch_drift(lp, C, alg, ro, Xo, **kw)
    assert stable.sum() >= 0.9 * 1024, stable.sum()
    for b in np.nonzero(stable)[0]:
        for k in ("status", "iterations", "attempts", "restarts"):
            assert res[b][k] == ro[b][k], (b, k, res[b][k], ro[b][k])
        assert rel(X[b], Xo[b]) <= max(1e-9, 100 * dx[b]), (b, rel(X[b], Xo[b]), dx[b])
    res = bs.solve(algorithm=alg, **CONST)
    X, Y = bs.solutions()
    bs.close()
    _, _, ro = oracle.solve_batch(lp, C, None, alg, **CONST)
    same = sum(res[b]["iterations"] == ro[b]["iterations"] for b in range(1024))
    assert same >= 0.6 * 1024, same
    for b in range(1024):
        assert res[b]["status"] == mp.LP_OPTIMAL and res[b]["rel_kkt"] <= 1e-4
        assert res[b]["attempts"] == res[b]["iterations"]
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert abs(res[b]["primal_objective"] - dp) <= 1e-3 * (1 + dp)
    # the point of the variant: no adaptive-step tail
    assert max(r["iterations"] for r in res) <= 4 * max(r["iterations"] for r in ro)


@pytest.mark.parametrize("alg", ALGS)
def test_constant_step_tiny_matches_generic_kernel(alg):
    """Register kernel (auto path) vs the generic per-instance kernel: the same
    arithmetic, reductions over a different lane/warp split (1-ulp differences in
    omega0 on a few instances), so identical over one check interval where stable."""
    lp, C = lpgen.g_grid(batch=256, seed=11)
    out = {}
    for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
        r64 = bs.solve(algorithm=alg, path=path, iteration_limit=64, eps_abs=0.0, eps_rel=0.0, **CONST)
        X64, _ = bs.solutions()
        res = bs.solve(algorithm=alg, path=path, **CONST)
        bs.close()
        out[path] = (r64, X64, res)
    (a64, XA, ra_), (b64, XB, rb_) = out[mp.PATH_AUTO], out[mp.PATH_INSTANCE]
    agree = sum(a64[b]["restarts"] == b64[b]["restarts"] and rel(XA[b], XB[b]) <= 1e-9 for b in range(256))
    assert agree >= 0.9 * 256, agree
    for b in range(256):
        assert ra_[b]["status"] == mp.LP_OPTIMAL and rb_[b]["status"] == mp.LP_OPTIMAL
        assert abs(ra_[b]["primal_objective"] - rb_[b]["primal_objective"]) <= 1e-3 * (1 + abs(rb_[b]["primal_objective"]))


@pytest.mark.parametrize("alg", ALGS)
def test_constant_step_grid_path(alg):
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=128, **CONST)
    ro, stable, drift = oracle_stability(lp, alg, **kw)
    rg = gpu_solve(lp, alg, path=mp.PATH_GRID, **kw)
    if stable:
        assert rg["restarts"] == ro["restarts"]
        assert rel(rg["x"], ro["x"]) <= max(1e-9, 100 * drift)
    rg = gpu_solve(lp, alg, path=mp.PATH_GRID, **CONST)
    assert rg["status"] == mp.LP_OPTIMAL and rg["rel_kkt"] <= 1e-4


@pytest.mark.parametrize("alg", ALGS)
def test_constant_step_dmma_path(alg):
    lp, C, Q, obj = lpgen.g_dense(40, 80, batch=16, seed=5)
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=64, **CONST)
    outs = []
    for path in (mp.PATH_DMMA, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
        res = bs.solve(algorithm=alg, path=path, **kw)
        X, _ = bs.solutions()
        bs.close()
        outs.append((res, X))
    Xo, _, ro = oracle.solve_batch(lp, C, Q, alg, **kw)
    for res, X in outs:
        for b in range(16):
            assert res[b]["attempts"] == 64
            if res[b]["restarts"] == ro[b]["restarts"]:
                assert rel(X[b], Xo[b]) <= 1e-8
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
    res = bs.solve(algorithm=alg, path=mp.PATH_DMMA, **CONST)
    bs.close()
    for b in range(16):
        assert res[b]["status"] == mp.LP_OPTIMAL
        assert abs(res[b]["primal_objective"] - obj[b]) <= 1e-3 * (1 + abs(obj[b]))


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 2, 4])
def test_constant_step_column_shards(alg, shards):
    """Column shards (reading 33): the power iteration on K~ split by columns -- each shard's
    slice of the unsharded start vector, K~x partials summed across shards, ||w||^2 summed across
    shards -- gives the oracle's step size to 1e-12 and its fixed-K trajectory."""
    lp = lpgen.g_rand(700, 9000, 30, seed=8)
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=64, **CONST)
    ro, stable, drift = oracle_stability(lp, alg, **kw)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards, axis="cols") as s:
        r = s.solve(algorithm=alg, **kw)
        x, y, _ = s.solution()
        assert abs(r["eta"] - oracle_eta(lp)) <= 1e-12 * oracle_eta(lp)
        if not stable:
            pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation")
        assert r["attempts"] == ro["attempts"] and r["restarts"] == ro["restarts"]
        tol = max(1e-9, 100 * drift)
        assert rel(x, ro["x"]) <= tol and rel(y, ro["y"]) <= tol
        r = s.solve(algorithm=alg, **CONST)
        assert r["status"] == mp.LP_OPTIMAL and r["rel_kkt"] <= 1e-4
        assert abs(r["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))


def test_constant_step_column_shards_nccl_one_rank():
    lp = lpgen.g_rand(700, 9000, 30, seed=8)
    comm = mp.nccl_comm_init(1, mp.nccl_unique_id(), 0)
    try:
        with mp.ShardedSolver(mp.local_cols(mp.Problem.from_lp(lp), 0, lp.n), axis="cols", n_global=lp.n,
                              comm=comm, rank=0, nranks=1) as s:
            a = s.solve(algorithm="r2", eps_abs=0.0, eps_rel=0.0, iteration_limit=64, **CONST)
            xa, _, _ = s.solution()
    finally:
        mp.nccl_comm_destroy(comm)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=1, axis="cols") as s:
        b = s.solve(algorithm="r2", eps_abs=0.0, eps_rel=0.0, iteration_limit=64, **CONST)
        xb, _, _ = s.solution()
    assert a["eta"] == b["eta"] and a["attempts"] == b["attempts"] and np.array_equal(xa, xb)


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 3])
def test_constant_step_sharded(alg, shards):
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=64, **CONST)
    ro, stable, drift = oracle_stability(lp, alg, **kw)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards) as s:
        r = s.solve(algorithm=alg, **kw)
        x, y, _ = s.solution()
        assert abs(r["eta"] - oracle_eta(lp)) <= 1e-12 * oracle_eta(lp)
        if stable:
            assert r["restarts"] == ro["restarts"] and rel(x, ro["x"]) <= max(1e-9, 100 * drift)
        r = s.solve(algorithm=alg, **CONST)
        assert r["status"] == mp.LP_OPTIMAL and r["rel_kkt"] <= 1e-4
