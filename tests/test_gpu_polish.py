"""GPU parity of feasibility polishing (DESIGN.md §3
reading 36) against the oracle on every solver path: the polished pair meets
eps_feas_polish on the ORIGINAL data (recomputed independently with the unscaled
K), the flags and counts follow the oracle, and the pair itself equals the
oracle's wherever the trajectories are well-posed (constant step: always on
these LPs; adaptive step: the sensitivity guard of test_gpu_parity.py)."""
import numpy as np
import pytest

import lpgen
import oracle
from tests.conftest import parity_log

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from tests.test_gpu_parity import rel  # noqa: E402

ALGS = ["ra", "r2"]
EPS_FP = 1e-6
POL = dict(feasibility_polishing=1)


def polished_ok(lp, x, y, eps=EPS_FP):
    k = oracle.kkt_original(lp, x, y)
    return (k["pres"] <= (1 + 1e-9) * eps * (1 + np.linalg.norm(lp.q)) and
            k["dres"] <= (1 + 1e-9) * eps * (1 + np.linalg.norm(lp.c)))


def gpu_single(lp, alg, **kw):
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        r = s.solve(algorithm=alg, **kw)
        x, y, lam = s.solution()
    r.update(x=x, y=y, lam=lam)
    return r


@pytest.mark.parametrize("rule", ["adaptive", "constant"])
@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("path", [mp.PATH_INSTANCE, mp.PATH_GRID])
def test_single_lp(path, alg, rule):
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    kw = dict(eps_abs=1e-2, eps_rel=1e-2, step_rule=rule)
    ro = oracle.solve(lp, alg, feasibility_polishing=True, **kw)
    rg = gpu_single(lp, alg, path=path, **POL, **kw)
    assert rg["status"] == ro["status"] == mp.LP_OPTIMAL
    assert rg["polish"] == ro["polish"] == 1
    assert polished_ok(lp, rg["x"], rg["y"])
    assert np.allclose(rg["lam"], lp.c - lp.dense_K().T @ rg["y"], atol=1e-9)
    k = oracle.kkt_original(lp, rg["x"], rg["y"])
    assert rg["primal_residual"] == pytest.approx(k["pres"], rel=1e-6, abs=1e-14)
    assert rg["dual_residual"] == pytest.approx(k["dres"], rel=1e-6, abs=1e-14)
    assert rg["primal_objective"] == pytest.approx(float(lp.c @ rg["x"]), rel=1e-12)
    if rule == "constant":  # well-posed trajectories: the same polished pair as the oracle
        assert rg["iterations"] == ro["iterations"]
        assert rel(rg["x"], ro["x"]) <= 1e-7 and rel(rg["y"], ro["y"]) <= 1e-7


@pytest.mark.parametrize("rule", ["adaptive", "constant"])
@pytest.mark.parametrize("alg", ALGS)
def test_c2_batch(alg, rule):
    """The C2 grid batch from eps 1e-3 (register kernel): every instance polished to
    1e-6 on the original data and still at the DP optimum to 1e-3."""
    lp, C = lpgen.g_grid(batch=256)
    kw = dict(eps_abs=1e-3, eps_rel=1e-3, step_rule=rule)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    res = bs.solve(algorithm=alg, **POL, **kw)
    X, Y = bs.solutions()
    bs.close()
    Xo, Yo, ro = oracle.solve_batch(lp, C, None, alg, feasibility_polishing=True, **kw)
    same = 0
    for b in range(256):
        assert res[b]["status"] == mp.LP_OPTIMAL and res[b]["polish"] == 1
        lb = lp.with_costs(c=C[b])
        assert polished_ok(lb, X[b], Y[b]), b
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert abs(res[b]["primal_objective"] - dp) <= 1e-2 * (1 + dp)
        if res[b]["iterations"] == ro[b]["iterations"]:
            same += 1
    assert same >= (0.95 if rule == "constant" else 0.5) * 256, same


@pytest.mark.parametrize("alg", ALGS)
def test_mixed_batch_polishes_only_optimal_instances(alg):
    """Unbounded instances keep their certificate rays and polish = 0."""
    lp = lpgen.g_infeasible("dual", 3, m1=10, m2=3, n=20, density=0.15)
    j = int(np.nonzero(~np.isfinite(lp.u))[0][0])
    C = np.tile(lp.c, (16, 1))
    C[::2, j] = np.abs(C[::2, j]) + 1.0
    for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
        res = bs.solve(algorithm=alg, path=path, iteration_limit=20000, step_rule="constant", **POL)
        X, Y = bs.solutions()
        bs.close()
        _, _, ro = oracle.solve_batch(lp, C, None, alg, iteration_limit=20000, step_rule="constant",
                                      feasibility_polishing=True)
        for b in range(16):
            assert res[b]["status"] == ro[b]["status"], (b, res[b]["status"], ro[b]["status"])
            assert res[b]["polish"] == ro[b]["polish"]
            if b % 2 == 0:
                assert res[b]["status"] == mp.LP_OPTIMAL and res[b]["polish"] == 1
                assert polished_ok(lp.with_costs(c=C[b]), X[b], Y[b])
            else:
                assert res[b]["status"] == mp.LP_DUAL_INFEASIBLE and res[b]["polish"] == 0
                assert abs(np.linalg.norm(X[b]) - 1) <= 1e-12


@pytest.mark.parametrize("alg", ALGS)
def test_dmma_dense_batch(alg):
    lp, C, Q, obj = lpgen.g_dense(40, 80, batch=16, seed=5)
    kw = dict(eps_abs=1e-3, eps_rel=1e-3)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
    res = bs.solve(algorithm=alg, path=mp.PATH_DMMA, **POL, **kw)
    X, Y = bs.solutions()
    bs.close()
    _, _, ro = oracle.solve_batch(lp, C, Q, alg, feasibility_polishing=True, **kw)
    capped = [b for b in range(16) if res[b]["polish"] == 2]
    parity_log(f"dmma_polish[{alg}]", polished=16 - len(capped), capped=len(capped), oracle_capped=sum(
        r["polish"] == 2 for r in ro), total=16)
    # a polish sub-solve may hit its 1e5-step cap (flag 2): the r2 adaptive-step polish
    # trajectories are chaotic (reading 30; the oracle needs 4e4-8e4 steps on two of these
    # instances and its FMA build differs), so a capped instance is counted, bounded, reported
    assert len(capped) <= (2 if alg == "r2" else 0), capped
    for b in range(16):
        assert res[b]["status"] == mp.LP_OPTIMAL and res[b]["polish"] in (1, 2)
        if res[b]["polish"] == 2:
            continue
        lb = lp.with_costs(c=C[b], q=Q[b])
        assert polished_ok(lb, X[b], Y[b])
        # polishing trades objective for feasibility (reported, not bounded: S:443); on these
        # LPs the oracle's polished primal objective moves up to 2% -- the GPU's must match it
        assert abs(res[b]["primal_objective"] - obj[b]) <= 5e-2 * (1 + abs(obj[b]))
        assert abs(res[b]["primal_objective"] - ro[b]["primal_objective"]) <= 1e-2 * (1 + abs(obj[b]))


def test_unfinished_polish_flag():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    r = gpu_single(lp, "ra", eps_abs=1e-2, eps_rel=1e-2, iteration_limit=192, eps_feas_polish=1e-14, **POL)
    ro = oracle.solve(lp, "ra", eps_abs=1e-2, eps_rel=1e-2, iteration_limit=192, feasibility_polishing=True,
                      eps_feas_polish=1e-14)
    assert r["status"] == ro["status"] == mp.LP_OPTIMAL and r["polish"] == ro["polish"] == 2
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=2) as s:
        r = s.solve(algorithm="ra", eps_abs=1e-2, eps_rel=1e-2, iteration_limit=192, eps_feas_polish=1e-14, **POL)
    assert r["status"] == mp.LP_OPTIMAL and r["polish"] == 2


@pytest.mark.parametrize("rule", ["adaptive", "constant"])
@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 2, 3])
def test_sharded(shards, alg, rule):
    """Polishing on the row-sharded engine (virtual shards on one GPU): the same two sub-solves
    and the same combination as every other path."""
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    kw = dict(eps_abs=1e-2, eps_rel=1e-2, step_rule=rule)
    ro = oracle.solve(lp, alg, feasibility_polishing=True, **kw)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards) as s:
        rg = s.solve(algorithm=alg, **POL, **kw)
        x, y, lam = s.solution()
    assert rg["status"] == ro["status"] == mp.LP_OPTIMAL
    assert rg["polish"] == ro["polish"] == 1
    assert polished_ok(lp, x, y)
    assert np.allclose(lam, lp.c - lp.dense_K().T @ y, atol=1e-9)
    k = oracle.kkt_original(lp, x, y)
    assert rg["primal_residual"] == pytest.approx(k["pres"], rel=1e-6, abs=1e-14)
    assert rg["dual_residual"] == pytest.approx(k["dres"], rel=1e-6, abs=1e-14)
    assert rg["primal_objective"] == pytest.approx(float(lp.c @ x), rel=1e-12)
    assert rg["dual_objective"] == pytest.approx(k["dobj"], rel=1e-9, abs=1e-12)
    if rule == "constant":  # well-posed trajectories: the same polished pair as the oracle
        assert rg["iterations"] == ro["iterations"]
        assert rel(x, ro["x"]) <= 1e-7 and rel(y, ro["y"]) <= 1e-7
    parity_log(f"sharded_polish[{shards},{alg},{rule}]", compared=1, total=1)


def test_no_polish_when_not_optimal():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    a = gpu_single(lp, "ra", eps_abs=1e-12, eps_rel=1e-12, iteration_limit=64, **POL)
    b = gpu_single(lp, "ra", eps_abs=1e-12, eps_rel=1e-12, iteration_limit=64)
    assert a["status"] == mp.LP_ITERATION_LIMIT and a["polish"] == 0 and np.array_equal(a["x"], b["x"])
    a = gpu_single(lp, "ra", eps_abs=1e-12, eps_rel=1e-12, iteration_limit=64, path=mp.PATH_GRID, **POL)
    assert a["status"] == mp.LP_ITERATION_LIMIT and a["polish"] == 0
