"""GPU parity of the partial-reflection variant of r2HPDHG (
DESIGN.md §3 reading 38): z <- a((1 + rho) PDHG(z) - rho z) + b z0 on every
solver path, against the oracle's `reflection` option."""
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


@pytest.mark.parametrize("rho", [0.0, 0.5])
@pytest.mark.parametrize("K", [1, 64])
@pytest.mark.parametrize("name,lp", list(small_lps()))
def test_fixed_K(rho, K, name, lp):
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=K, reflection=rho)
    ro, stable, drift = oracle_stability(lp, "r2", **kw)
    rg = gpu_solve(lp, "r2", **kw)
    if not stable:
        pytest.skip("ill-conditioned at this K")
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rel(rg["x"], ro["x"]) <= max(1e-9, 100 * drift)


@pytest.mark.parametrize("path", [mp.PATH_AUTO, mp.PATH_INSTANCE])
def test_c2_batch_removes_the_adaptive_tail(path):
    """rho = 0.8 with the adaptive step: K = 64 parity on every stable instance, then full
    solves all OPTIMAL at the DP optimum with no ~1e4-iteration tail (reading 38)."""
    lp, C = lpgen.g_grid(batch=1024)
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=64, reflection=0.8)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    res = bs.solve(algorithm="r2", path=path, **kw)
    X, _ = bs.solutions()
    Xo, _, ro = oracle.solve_batch(lp, C, None, "r2", **kw)
    stable, dx, _ = batch_drift(lp, C, "r2", ro, Xo, **kw)
    for b in np.nonzero(stable)[0]:
        assert res[b]["attempts"] == ro[b]["attempts"] and rel(X[b], Xo[b]) <= max(1e-9, 100 * dx[b])
    res = bs.solve(algorithm="r2", path=path, reflection=0.8)
    bs.close()
    assert res["iterations"].max() <= 2000, res["iterations"].max()
    for b in range(1024):
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert res[b]["status"] == mp.LP_OPTIMAL and abs(res[b]["primal_objective"] - dp) <= 1e-3 * (1 + dp)


def test_grid_dmma_sharded_paths():
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=64, reflection=0.5, step_rule="constant")
    ro = oracle.solve(lp, "r2", **kw)
    rg = gpu_solve(lp, "r2", path=mp.PATH_GRID, **kw)
    assert rg["restarts"] == ro["restarts"] and rel(rg["x"], ro["x"]) <= 1e-9
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=3) as s:
        rs = s.solve(algorithm="r2", **kw)
        xs, _, _ = s.solution()
    assert rs["restarts"] == ro["restarts"] and rel(xs, ro["x"]) <= 1e-9
    dl, C, Q, _ = lpgen.g_dense(40, 80, batch=16, seed=5)
    bs = mp.BatchSolver(mp.Problem.from_lp(dl), C, Q)
    res = bs.solve(algorithm="r2", path=mp.PATH_DMMA, **kw)
    X, _ = bs.solutions()
    bs.close()
    Xo, _, rob = oracle.solve_batch(dl, C, Q, "r2", **kw)
    for b in range(16):
        if res[b]["restarts"] == rob[b]["restarts"]:
            assert rel(X[b], Xo[b]) <= 1e-8


def test_invalid_reflection_is_rejected():
    with mp.Solver(mp.Problem.from_lp(lpgen.tiny_spec())) as s:
        with pytest.raises(mp.LpError):
            s.solve(algorithm="r2", reflection=1.5)
