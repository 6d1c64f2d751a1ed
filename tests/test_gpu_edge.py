"""Edge cases of the batched paths against the oracle and closed forms (the parity bar of
the task: empty and ragged inputs, maximum sizes, degenerate cases): a 65 536-instance batch
(many scheduler waves), box-only LPs (m = 0, closed-form optimum), one-variable LPs, zero
rows / columns in K, device-memory warm starts, lp_update_batch, and invalid batch shapes."""
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

DEV = torch.device("cuda", 0)


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_max_batch_65536(alg):
    """64x the C2 batch on the register kernel: every instance OPTIMAL at its DP optimum; a
    128-instance sample held to fixed-K parity on its count-stable members."""
    lp, C = lpgen.g_grid(batch=65536, seed=21)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp).to(DEV), torch.as_tensor(C, device=DEV))
    res = bs.solve(algorithm=alg, step_rule="constant")
    assert (res["status"] == mp.LP_OPTIMAL).all() and (res["rel_kkt"] <= 1e-4).all()
    dp = np.array([lpgen.grid_dp_optimum(5, C[b]) for b in range(0, 65536, 97)])
    got = res["primal_objective"][::97]
    assert np.all(np.abs(got - dp) <= 1e-3 * (1 + dp))
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=64, step_rule="constant")
    res = bs.solve(algorithm=alg, **kw)
    X, _ = bs.solutions()
    bs.close()
    idx = np.arange(0, 65536, 512)
    Xo, _, ro = oracle.solve_batch(lp, C[idx], None, alg, **kw)
    stable, dx, _ = batch_drift(lp, C[idx], alg, ro, Xo, **kw)
    assert stable.sum() >= 0.9 * len(idx)
    for t in np.nonzero(stable)[0]:
        b = idx[t]
        assert res[b]["attempts"] == ro[t]["attempts"] and rel(X[b], Xo[t]) <= max(1e-9, 100 * dx[t])


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_box_only_batch(alg):
    """m = 0: min c'x over a box has the closed form x_j = l_j if c_j > 0, u_j if c_j < 0."""
    rng = np.random.default_rng(3)
    n = 33
    lp = lpgen.stack(rng.normal(size=n), l=-rng.uniform(0.5, 2, n), u=rng.uniform(0.5, 2, n))
    C = rng.normal(size=(200, n))
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    res = bs.solve(algorithm=alg, eps_abs=1e-10, eps_rel=1e-10)
    X, _ = bs.solutions()
    bs.close()
    want = np.where(C > 0, lp.l, lp.u)
    assert (res["status"] == mp.LP_OPTIMAL).all()
    assert np.allclose(X, want, rtol=0, atol=1e-8)


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_one_variable_lps(alg):
    """n = 1: min c x s.t. x >= h, 0 <= x <= 5 -> x = max(h, 0) for c > 0."""
    lp = lpgen.stack([1.0], G=[[1.0]], h=[1.0], l=[0.0], u=[5.0])
    Q = np.array([[h] for h in np.linspace(-1.0, 4.0, 11)])
    C = np.ones((11, 1))
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
    res = bs.solve(algorithm=alg, eps_abs=1e-10, eps_rel=1e-10)
    X, _ = bs.solutions()
    bs.close()
    assert (res["status"] == mp.LP_OPTIMAL).all()
    assert np.allclose(X[:, 0], np.maximum(Q[:, 0], 0.0), atol=1e-8)


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_zero_row_and_column(alg):
    """An all-zero row (h <= 0, so satisfiable) and an all-zero column (a pure box variable)."""
    rng = np.random.default_rng(9)
    G = rng.normal(size=(6, 8)) * (rng.random((6, 8)) < 0.6)
    G[2, :] = 0.0
    G[:, 5] = 0.0
    x0 = rng.uniform(0.2, 0.8, size=8)
    h = G @ x0 - 0.1
    h[2] = -1.0
    lp = lpgen.stack(rng.normal(size=8), G=G, h=h, l=np.zeros(8), u=np.ones(8))
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=64)
    ro = oracle.solve(lp, alg, **kw)
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        rg = s.solve(algorithm=alg, **kw)
        x, _, _ = s.solution()
    assert rg["attempts"] == ro["attempts"] and rel(x, ro["x"]) <= 1e-9
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        rg = s.solve(algorithm=alg, eps_abs=1e-9, eps_rel=1e-9)
        x, _, _ = s.solution()
    assert rg["status"] == mp.LP_OPTIMAL
    assert x[5] == pytest.approx(0.0 if lp.c[5] > 0 else 1.0, abs=1e-7)   # the free-standing column


def test_device_warm_start_and_update_batch():
    """Warm starts from device memory equal host ones bitwise; lp_update_batch then solve equals
    a fresh handle bitwise."""
    lp, C = lpgen.g_grid(batch=128, seed=4)
    rng = np.random.default_rng(1)
    X0, Y0 = rng.uniform(0, 1, size=(128, lp.n)), rng.normal(size=(128, lp.m))
    a = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    ra_ = a.solve(X0, Y0, algorithm="r2")
    Xa, _ = a.solutions()
    a.close()
    b = mp.BatchSolver(mp.Problem.from_lp(lp).to(DEV), torch.as_tensor(C, device=DEV))
    rb = b.solve(torch.as_tensor(X0, device=DEV), torch.as_tensor(Y0, device=DEV), algorithm="r2")
    Xb, _ = b.solutions()
    C2 = C[::-1].copy()
    b.update(torch.as_tensor(C2, device=DEV))
    ru = b.solve(algorithm="ra")
    Xu, _ = b.solutions()
    b.close()
    assert np.array_equal(Xa, Xb) and np.array_equal(ra_["attempts"], rb["attempts"])
    f = mp.BatchSolver(mp.Problem.from_lp(lp), C2)
    rf = f.solve(algorithm="ra")
    Xf, _ = f.solutions()
    f.close()
    assert np.array_equal(Xu, Xf) and np.array_equal(ru["attempts"], rf["attempts"])


def test_invalid_batch_shapes():
    lp, C = lpgen.g_grid(batch=4)
    with pytest.raises(mp.LpError):
        mp.BatchSolver(mp.Problem.from_lp(lp), C[:0])            # batch of 0
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), None, np.tile(lp.q, (4, 1)))
    with pytest.raises(mp.LpError):
        bs.update(C)                                             # the handle shares one c
    bs.close()


def test_division_fast_path_is_bitwise_ieee():
    """div_rn_fast (common.cuh), used for eta_bar = M / (2|I|) and eta / (W + eta) in the
    latency-bound kernels, is bit-identical to IEEE a / b whenever its range test passes."""
    for seed in (1, 2):
        mism, slow = mp.selftest_division(1 << 26, seed)
        assert mism == 0, mism
        assert 0 < slow < (1 << 26) // 2, slow      # the special / extreme operands take the slow path


def test_update_batch_validates_and_sharded_handles_refuse_batch_calls():
    """lp_update_batch checks the new costs like lp_create (LP_ERR_NAN) and is synchronous;
    calls that have no meaning on a row-sharded handle return LP_ERR_UNSUPPORTED instead of
    silently doing nothing."""
    lp, C = lpgen.g_grid(batch=8)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    bs.solve(algorithm="ra")
    bad = C.copy()
    bad[3, 5] = np.nan
    with pytest.raises(mp.LpError) as e:
        bs.update(bad)
    assert e.value.code == -3
    with pytest.raises(mp.LpError) as e:          # no solution is kept after a rejected update
        bs.solutions()
    assert e.value.code == -9
    bs.update(C)
    res = bs.solve(algorithm="ra")
    assert all(r["status"] == mp.LP_OPTIMAL for r in res)
    bs.close()
    with mp.ShardedSolver(mp.Problem.from_lp(lpgen.g_rand(50, 100, 10, seed=1)), virtual_shards=2) as s:
        for call in (lambda: mp.lib().lp_get_solutions(s._h, None, None, 0),
                     lambda: mp.lib().lp_get_scaling(s._h, None, None, 0),
                     lambda: mp.lib().lp_update_batch(s._h, None, None, 0)):
            assert call() == -10
