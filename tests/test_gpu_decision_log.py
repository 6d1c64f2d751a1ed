"""The GPU decision log (lp_set_decision_log, grid path) against the oracle's own log
(floating-point differences "can accumulate over time").

Where GPU and oracle agree on the counts, every logged decision must agree: the same accept /
reject sequence, the same restart flags and outcomes, eta and eta_bar equal to rounding.  Where
they part ways, the first decision that differs must be a near tie in the oracle's own log --
eta within a hair of eta_bar, or a restart metric within a hair of one of its thresholds --
which is what rounding-order noise can flip; a decision flipped with a wide margin is a bug."""
import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from tests.conftest import parity_log  # noqa: E402
from tests.test_gpu_grid import CASES  # noqa: E402

ALGS = ["ra", "r2"]
# restart thresholds of the contract (c.2 step 5): sufficient 0.2 ref, necessary 0.8 ref
BETA_SUFF, BETA_NEC = 0.2, 0.8


def gpu_logged(lp, alg, **kw):
    with mp.Solver(mp.Problem.from_lp(lp).to("cuda")) as s:
        s.set_decision_log(att_cap=20000, chk_cap=1000)
        r = s.solve(algorithm=alg, path=mp.PATH_GRID, **kw)
        att, chk = s.decision_log()
    return r, att, chk


def attempt_margin(row):
    """Relative distance of the accept test eta <= eta_bar from its tie."""
    eta, eb = row[2], row[3]
    return abs(eta - eb) / max(abs(eb), 1e-300) if np.isfinite(eb) else np.inf


def check_margin(row):
    """Relative distance of the restart metric from the nearest threshold it is compared with."""
    _, metric, ref, last = row[:4]
    cands = [abs(metric - BETA_SUFF * ref), abs(metric - BETA_NEC * ref)]
    if np.isfinite(last):
        cands.append(abs(metric - last))
    return min(cands) / max(abs(ref), abs(metric), 1e-300)


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("name,lp", CASES)
def test_decision_log_matches_oracle(alg, name, lp):
    ro = oracle.solve(lp, alg, log_capacity=20000)
    rg, att, chk = gpu_logged(lp, alg)
    oa, oc = ro["att_log"], ro["chk_log"]
    assert len(att) == rg["attempts"] and len(chk) >= 1
    assert np.array_equal(att[:, 0], np.arange(1, len(att) + 1))       # every attempt logged, in order
    assert int(np.sum(att[:, 1])) == rg["iterations"]                    # accepted rows = iterations
    assert np.all(chk[:, 0] > 0) and np.all(np.diff(chk[:, 0]) > 0)
    n = min(len(att), len(oa))
    diff_a = np.nonzero(att[:n, 1] != oa[:n, 1])[0]
    nc = min(len(chk), len(oc))
    diff_c = np.nonzero((chk[:nc, 4] != oc[:nc, 4]) | (chk[:nc, 5] != oc[:nc, 5]))[0]
    if rg["attempts"] == ro["attempts"] and rg["restarts"] == ro["restarts"] and not len(diff_a) and not len(diff_c):
        # same decisions: every logged value agrees to within the rounding amplification the
        # oracle itself shows -- its FMA-contracted build (an equally valid evaluation order,
        # reading 27) logs the same decisions with values that drift by `amp`; eta_bar = M / 2|I|
        # carries the cancellation in I, so late attempts drift most
        assert len(att) == len(oa) and len(chk) == len(oc)
        rf = oracle.solve(lp, alg, log_capacity=20000, fma=True)
        fa, fc = rf["att_log"], rf["chk_log"]
        same_f = len(fa) == len(oa) and np.array_equal(fa[:, 1], oa[:, 1])
        amp = float(np.max(np.abs(fa[:, 2:] - oa[:, 2:]) / np.maximum(np.abs(oa[:, 2:]), 1e-300))) if same_f else 1e-4
        tol = max(1e-10, 100 * amp)
        np.testing.assert_allclose(att[:, 2:], oa[:, 2:], rtol=tol)
        fin = np.isfinite(oc[:, 1:4])
        np.testing.assert_allclose(chk[:, 1:4][fin], oc[:, 1:4][fin], rtol=tol)
        # the first attempts, before any amplification, agree to a few ulps
        np.testing.assert_allclose(att[:8, 2:], oa[:8, 2:], rtol=1e-12)
        gdev = float(np.max(np.abs(att[:, 2:] - oa[:, 2:]) / np.maximum(np.abs(oa[:, 2:]), 1e-300)))
        parity_log(f"decision_log[{name},{alg}]", same=1, attempts=len(att), checks=len(chk), gpu_dev=gdev,
                   fma_dev=amp)
        return
    # the trajectories part: the first differing decision must be a near tie in the oracle
    ja = int(diff_a[0]) if len(diff_a) else None
    jc = int(diff_c[0]) if len(diff_c) else None
    k_a = np.cumsum(oa[:, 1])[ja] if ja is not None else np.inf      # accepted steps at that attempt
    rows = None
    bound = 1e-2
    if jc is not None and oc[jc, 0] <= k_a:
        k = int(oc[jc, 0])
        if chk[jc, 5] != oc[jc, 5]:
            # the termination test went the other way: its margin is the distance of the oracle's
            # relative KKT error at this check from the tolerance (pass <=> rel_kkt <= 1e-4 here),
            # judged against how far the oracle's own FMA-contracted build moves that error by k
            rk = oracle.solve(lp, alg, iteration_limit=k, eps_abs=0.0, eps_rel=0.0)["rel_kkt"]
            rkf = oracle.solve(lp, alg, iteration_limit=k, eps_abs=0.0, eps_rel=0.0, fma=True)["rel_kkt"]
            margin = abs(rk - 1e-4) / 1e-4
            bound = max(1e-2, 10 * abs(rkf - rk) / rk)
            where = f"termination test at k={k}"
        else:
            margin = check_margin(oc[jc])
            where = f"restart test at k={k}"
        rows = (oc[jc].tolist(), chk[jc].tolist())
    elif ja is not None:
        margin = attempt_margin(oa[ja])
        where = f"line search at j={ja + 1}"
        if not np.isfinite(oa[ja, 3]):
            # I = <dy, K dx> is exactly 0 in the oracle (eta_bar = M / 2|I| = inf: a converged or
            # degenerate step, M / I a 0/0 form) and rounding-level on the GPU: the tie is the
            # degeneracy itself
            margin = 0.0
            where += " (I = 0 in the oracle)"
        rows = (oa[ja].tolist(), att[ja].tolist())
    else:   # every common decision agrees; one log is a prefix of the other
        margin = check_margin(oc[nc - 1]) if nc else 0.0
        where = "termination"
    parity_log(f"decision_log[{name},{alg}]", same=0, first_divergence=where, margin=margin, bound=bound,
               oracle_row=str(rows[0]) if rows else "", gpu_row=str(rows[1]) if rows else "")
    assert margin <= bound, (where, margin, bound, rows)


def test_decision_log_off_and_unsupported():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    with mp.Solver(mp.Problem.from_lp(lp).to("cuda")) as s:
        s.set_decision_log(att_cap=100, chk_cap=10)
        with pytest.raises(mp.LpError) as e:
            s.solve(algorithm="r2", path=mp.PATH_INSTANCE)
        assert e.value.code == -10
        r = s.solve(algorithm="r2", path=mp.PATH_GRID)
        att, chk = s.decision_log()
        assert len(att) == min(100, r["attempts"]) and chk[-1, 5] == 1   # capacity respected; optimal
        s.set_decision_log(att_cap=0, chk_cap=0)
        assert s.solve(algorithm="r2")["status"] == mp.LP_OPTIMAL         # log off: any path again
