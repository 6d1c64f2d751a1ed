"""GPU parity of the shared-dense-K tensor-core path (DMMA, SURVEY §8(a) a12,
config C3) against the CPU oracle, through the C ABI."""
import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from tests.test_gpu_parity import batch_drift, rel  # noqa: E402

ALGS = ["ra", "r2"]


def dmma_batch(lp, C, Q, alg, **kw):
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
    res = bs.solve(algorithm=alg, path=mp.PATH_DMMA, **kw)
    X, Y = bs.solutions()
    bs.close()
    return res, X, Y


CASES = [("small", 60, 90, 20, 5), ("C3-shape", 200, 400, 16, 3), ("odd", 37, 53, 9, 7)]


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 2, 64])
@pytest.mark.parametrize("name,m,n,B,seed", CASES)
def test_dmma_fixed_K(alg, K, name, m, n, B, seed):
    lp, C, Q, obj = lpgen.g_dense(m, n, batch=B, seed=seed)
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=K)
    res, X, Y = dmma_batch(lp, C, Q, alg, **kw)
    Xo, Yo, ro = oracle.solve_batch(lp, C, Q, alg, **kw)
    stable, dx = batch_drift_q(lp, C, Q, alg, ro, Xo, **kw)
    assert stable.sum() >= 0.75 * B, stable.sum()
    for b in np.nonzero(stable)[0]:
        for k in ("status", "iterations", "attempts", "restarts"):
            assert res[b][k] == ro[b][k], (b, k, res[b][k], ro[b][k])
        tol = max(1e-9, 100 * dx[b])
        assert rel(X[b], Xo[b]) <= tol, (b, rel(X[b], Xo[b]), dx[b])
        assert rel(Y[b], Yo[b]) <= max(tol, 1e-8)


def batch_drift_q(lp, C, Q, alg, ro, X, **kw):
    keys = ("status", "iterations", "attempts", "restarts")
    from tests.test_gpu_parity import ulp_perturb
    B = C.shape[0]
    stable = np.ones(B, bool)
    dx = np.zeros(B)
    for seed in (1, 2):
        Xp, _, rp = oracle.solve_batch(lp, ulp_perturb(C, seed), Q, alg, **kw)
        for b in range(B):
            stable[b] &= all(rp[b][k] == ro[b][k] for k in keys)
            dx[b] = max(dx[b], rel(Xp[b], X[b]))
    return stable, dx


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("name,m,n,B,seed", CASES)
def test_dmma_full_solve(alg, name, m, n, B, seed):
    lp, C, Q, obj = lpgen.g_dense(m, n, batch=B, seed=seed)
    res, X, Y = dmma_batch(lp, C, Q, alg)
    Xo, Yo, ro = oracle.solve_batch(lp, C, Q, alg)
    same = 0
    for b in range(B):
        assert res[b]["status"] == mp.LP_OPTIMAL and res[b]["rel_kkt"] <= 1e-4, (b, res[b])
        assert abs(res[b]["primal_objective"] - obj[b]) <= 1e-3 * (1 + abs(obj[b]))
        k = oracle.kkt_original(lp.with_costs(c=C[b], q=Q[b]), X[b], Y[b])
        assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(Q[b]))
        assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(C[b]))
        same += res[b]["attempts"] == ro[b]["attempts"]
    assert same >= B // 2, same


def test_dmma_matches_per_instance_path():
    lp, C, Q, obj = lpgen.g_dense(60, 90, batch=24, seed=11)
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=64, algorithm="ra")
    a = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
    ra = a.solve(path=mp.PATH_DMMA, **kw)
    Xa, _ = a.solutions()
    a.close()
    b = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
    rb = b.solve(path=mp.PATH_INSTANCE, **kw)
    Xb, _ = b.solutions()
    b.close()
    agree = sum(ra[i]["attempts"] == rb[i]["attempts"] and rel(Xa[i], Xb[i]) <= 1e-9 for i in range(24))
    assert agree >= 20, agree
