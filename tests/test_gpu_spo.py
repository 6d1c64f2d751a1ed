"""GPU parity of the SPO+ layer (PAPER.md Eq. (spo+ loss)
P:76-78, Eq. (spo+ gradient) P:80-82, listing P:198-215) against the oracle's
spo_plus on paper-shaped batches: Warcraft-shaped 8-connected grids (k = 12,
batch 70) and dense knapsack LPs."""
import numpy as np
import pytest
from scipy.optimize import linprog

import lpgen
import oracle
from oracle.spo import spo_plus

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from paper_2412_09734_b200.spo import spo_plus_loss  # noqa: E402


def true_solutions(lp, C):
    """x*(c_b) by HiGHS (a library LP solver), and c_b'x*(c_b)."""
    K = lp.dense_K()
    X = []
    for c in C:
        r = linprog(c, A_ub=-K[: lp.m1] if lp.m1 else None, b_ub=-lp.q[: lp.m1] if lp.m1 else None,
                    A_eq=K[lp.m1:] if lp.m2 else None, b_eq=lp.q[lp.m1:] if lp.m2 else None,
                    bounds=list(zip(lp.l, lp.u)), method="highs-ds")
        X.append(r.x)
    X = np.array(X)
    return X, np.sum(C * X, axis=1)


def warcraft_batch(k=12, B=70, seed=1):
    lp = lpgen.warcraft_lp(k)
    Ct = lpgen.warcraft_costs(k, B, seed)
    Cp = Ct * np.random.default_rng(seed + 50).uniform(0.5, 1.5, size=Ct.shape)   # a predictor's output
    Xt, ot = true_solutions(lp, Ct)
    return lp, Cp, Ct, Xt, ot


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_warcraft_batch_matches_oracle(alg):
    lp, Cp, Ct, Xt, ot = warcraft_batch()
    kw = dict(eps_abs=1e-4, eps_rel=1e-4, step_rule="constant")
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), Ct)
    loss, grad, res = bs.spo_plus(Cp, Ct, Xt, ot, algorithm=alg, **kw)
    X, _ = bs.solutions()
    bs.close()
    lo, go, Xo, _, ro = spo_plus(lp, Cp, Ct, Xt, ot, alg, **kw)
    assert all(r["status"] == mp.LP_OPTIMAL for r in res)
    same = 0
    for b in range(70):
        if res[b]["iterations"] == ro[b]["iterations"]:
            same += 1
            assert abs(loss[b] - lo[b]) <= 1e-7 * (1 + abs(lo[b])), (b, loss[b], lo[b])
            assert np.abs(grad[b] - go[b]).max() <= 1e-6
        # any eps-optimal inner solution: the loss within the inner solve's objective tolerance
        assert abs(loss[b] - lo[b]) <= 1e-3 * (1 + abs(ot[b]))
        assert np.allclose(grad[b], 2 * (Xt[b] - X[b]), atol=0, rtol=0)
        assert np.all(np.abs(grad[b]) <= 2 + 1e-6)
    assert same >= 0.9 * 70, same


def test_autograd_layer_on_device_and_warm_start():
    """The torch layer: loss = batch mean, backward = grad / B; a warm-started second step
    (predictions moved slightly, as between epochs) needs fewer iterations."""
    lp, Cp, Ct, Xt, ot = warcraft_batch(seed=4)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.as_tensor(a, device=dev)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp).to(dev), T(Ct))
    pred = T(Cp).requires_grad_(True)
    loss = spo_plus_loss(pred, T(Ct), T(Xt), T(ot), bs, algorithm="r2")
    loss.backward()
    l_ref, g_ref, r_cold = bs.spo_plus(T(Cp), T(Ct), T(Xt), T(ot), algorithm="r2")
    assert abs(loss.item() - l_ref.mean().item()) <= 1e-12 * (1 + abs(loss.item()))
    assert torch.allclose(pred.grad, g_ref / 70, rtol=0, atol=1e-15)
    Cp2 = Cp * np.random.default_rng(9).uniform(0.98, 1.02, size=Cp.shape)
    _, _, r_warm = bs.spo_plus(T(Cp2), T(Ct), T(Xt), T(ot), algorithm="r2", warm=True)
    bs2 = mp.BatchSolver(mp.Problem.from_lp(lp).to(dev), T(Ct))
    _, _, r_cold2 = bs2.spo_plus(T(Cp2), T(Ct), T(Xt), T(ot), algorithm="r2")
    bs.close(); bs2.close()
    assert all(r["status"] == mp.LP_OPTIMAL for r in r_warm)
    assert r_warm["iterations"].sum() < r_cold2["iterations"].sum(), (r_warm["iterations"].sum(),
                                                                      r_cold2["iterations"].sum())


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_dense_knapsack_batch(alg):
    """Shared dense K (DMMA path for batches >= 8)."""
    lp = lpgen.knapsack_lp(400, 10, seed=3)
    Ct = lpgen.knapsack_values(400, 16, seed=4, noise=0.5)
    Cp = Ct * np.random.default_rng(5).uniform(0.7, 1.3, size=Ct.shape)
    Xt, ot = true_solutions(lp, Ct)
    kw = dict(eps_abs=1e-4, eps_rel=1e-4)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), Ct)
    loss, grad, res = bs.spo_plus(Cp, Ct, Xt, ot, algorithm=alg, path=mp.PATH_DMMA, **kw)
    bs.close()
    lo, go, _, _, ro = spo_plus(lp, Cp, Ct, Xt, ot, alg, **kw)
    for b in range(16):
        assert res[b]["status"] == mp.LP_OPTIMAL
        assert loss[b] >= -1e-3 * (1 + abs(ot[b]))                  # SPO+ >= 0, to the inner tolerance
        assert abs(loss[b] - lo[b]) <= 1e-3 * (1 + abs(ot[b]))


def test_shared_cost_handle_is_rejected():
    lp, Cp, Ct, Xt, ot = warcraft_batch(k=4, B=3)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), None, np.tile(lp.q, (3, 1)))
    with pytest.raises(mp.LpError):
        bs.spo_plus(Cp, Ct, Xt, ot)
    bs.close()
