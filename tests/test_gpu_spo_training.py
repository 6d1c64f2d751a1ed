"""SPEC acceptance #9, the desk-scale analogue of the paper's training curves
(Fig. 2): a linear predictor trained by plain gradient descent on the SPO+ loss
(this library's layer: inner LPs solved by the CUDA path, warm-started across epochs) over 50
synthetic knapsack samples (N = 20, d = 3, noiseless polynomial ground truth) must cut the
training loss by >= 50% and reach a normalized test regret below 5% within 30 epochs (eps 1e-4).
Normalized regret (test-only; SURVEY §2 keeps it out of the product): sum_i c_i'(x(c^_i) -
x*(c_i)) / sum_i |c_i'x*(c_i)| for the minimisation form."""
import numpy as np
import pytest

import lpgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from paper_2412_09734_b200.spo import spo_plus_loss  # noqa: E402

N, D, P = 20, 3, 5


def dataset(n_samples, seed, B):
    """Features f ~ N(0, I_5); values c = [((B f)/sqrt5 + 3)^4 + 1] / 3.5^4 (PyEPO polynomial,
    noiseless); minimisation costs -c."""
    rng = np.random.default_rng(seed)
    F = rng.normal(size=(n_samples, P))
    V = (((F @ B.T) / np.sqrt(P) + 3.0) ** 4 + 1.0) / 3.5 ** 4
    return F, -V


def test_spo_plus_training_reduces_loss_and_regret():
    dev = torch.device("cuda", 0)
    lp = lpgen.knapsack_lp(N, D, seed=7, capacity=30.0, dense=False)
    B = (np.random.default_rng(8).uniform(size=(N, P)) < 0.5).astype(np.float64)
    Ftr, Ctr = dataset(50, 9, B)
    Fte, Cte = dataset(50, 10, B)
    T = lambda a: torch.as_tensor(a, device=dev)
    prob = mp.Problem.from_lp(lp).to(dev)
    opts = dict(algorithm="r2", step_rule="constant", eps_abs=1e-4, eps_rel=1e-4)

    def solve(C):
        bs = mp.BatchSolver(prob, T(C))
        res = bs.solve(**opts)
        X, _ = bs.solutions(memory=mp.LP_DEVICE)
        bs.close()
        assert (res["status"] == mp.LP_OPTIMAL).all()
        return X

    Xtr = solve(Ctr)
    otr = (T(Ctr) * Xtr).sum(dim=1)
    Xte = solve(Cte)
    ote = (T(Cte) * Xte).sum(dim=1)

    torch.manual_seed(0)
    W = (0.1 * torch.randn(N, P, dtype=torch.float64, device=dev)).requires_grad_(True)
    b = torch.zeros(N, dtype=torch.float64, device=dev, requires_grad=True)
    layer = mp.BatchSolver(prob, T(Ctr))
    losses = []
    for epoch in range(30):
        pred = T(Ftr) @ W.T + b
        loss = spo_plus_loss(pred, T(Ctr), Xtr, otr, layer, warm=epoch > 0, **opts)
        W.grad = None
        b.grad = None
        loss.backward()
        with torch.no_grad():
            W -= 0.5 * W.grad
            b -= 0.5 * b.grad
        losses.append(loss.item())
    layer.close()

    with torch.no_grad():
        pred_te = (T(Fte) @ W.T + b).cpu().numpy()
    Xhat = solve(pred_te)
    regret = float(((T(Cte) * Xhat).sum(dim=1) - ote).sum() / ote.abs().sum())
    assert losses[-1] <= 0.5 * losses[0], losses
    assert regret < 0.05, regret
