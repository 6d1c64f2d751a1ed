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


def probe_logs(lp, alg, cap):
    """The oracle's own rounding sensitivity: its FMA-contracted build (reading 27) and a solve on
    c perturbed by one ulp per entry (random signs) -- equally valid roundings of the contract."""
    rf = oracle.solve(lp, alg, log_capacity=cap, fma=True)
    sgn = np.random.default_rng(11).choice([-1.0, 1.0], size=lp.n)
    cp = lp.c + sgn * np.spacing(lp.c)
    ru = oracle.solve(lp.with_costs(c=cp), alg, log_capacity=cap)
    return [rf["att_log"], ru["att_log"]]


def eta_drift(a, o, w):
    """Largest relative difference of the tried step sizes eta over the first w attempts."""
    if w <= 0:
        return 0.0
    return float(np.max(np.abs(a[:w, 2] - o[:w, 2]) / np.maximum(np.abs(o[:w, 2]), 1e-300)))


def compare_logs(lp, alg, rg, att, chk, ro, name):
    """Same decisions: every logged value within 100x the FMA build's own drift.  Diverging
    decisions: the first one must be a near tie in the oracle's log.  Returns the parity record."""
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
        # (eta is compared: eta_bar = M / 2|I| magnifies the cancellation in I without bound)
        assert len(att) == len(oa) and len(chk) == len(oc)
        amp = 0.0
        for pa in probe_logs(lp, alg, len(oa) + 64):
            w = min(len(pa), len(oa))
            d = np.nonzero(pa[:w, 1] != oa[:w, 1])[0]
            amp = max(amp, eta_drift(pa, oa, int(d[0]) if len(d) else w))
        gdev = eta_drift(att, oa, len(oa))
        assert gdev <= max(1e-6, 100 * amp), (name, gdev, amp)
        # the first attempts, before any amplification, agree to rounding (reduction order differs)
        np.testing.assert_allclose(att[:8, 2:], oa[:8, 2:], rtol=1e-9)
        return dict(same=1, attempts=len(att), checks=len(chk), gpu_drift=gdev, probe_drift=amp)
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
    rec = dict(same=0, first_divergence=where, margin=margin, bound=bound,
               oracle_row=str(rows[0]) if rows else "", gpu_row=str(rows[1]) if rows else "")
    if margin <= bound:
        return rec
    # not a tie at the split: the trajectories drifted apart continuously before it (the
    # contract's dynamics amplify rounding, reading 30).  Then the GPU's drift from the oracle over
    # the common decisions must stay within what an equally valid rounding of the oracle itself
    # produces there: the FMA-contracted build's drift on the same attempts (x100, the parity bar)
    end = ja if ja is not None else n
    gdev = eta_drift(att, oa, end)
    fdev, split = 0.0, end
    for pa in probe_logs(lp, alg, len(oa) + 64):
        w = min(end, len(pa))
        d = np.nonzero(pa[:w, 1] != oa[:w, 1])[0]
        w = int(d[0]) if len(d) else w            # a probe's own decisions may part earlier
        split = min(split, w)
        fdev = max(fdev, eta_drift(pa, oa, w))
    rec.update(gpu_drift=gdev, probe_drift=fdev, probe_split=int(split))
    assert split < end or gdev <= max(1e-6, 100 * fdev), (name, rec)
    return rec


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("name,lp", CASES)
def test_decision_log_matches_oracle(alg, name, lp):
    ro = oracle.solve(lp, alg, log_capacity=20000)
    rg, att, chk = gpu_logged(lp, alg)
    parity_log(f"decision_log[{name},{alg}]", **compare_logs(lp, alg, rg, att, chk, ro, name))


@pytest.mark.parametrize("alg", ALGS)
def test_c2_batch_divergences_are_near_ties(alg):
    """The register kernel's log of one C2 instance (lp_set_decision_log_instance): on the
    instances whose counts differ from the oracle's, the first differing decision is a near tie;
    on one instance that agrees, every logged value agrees.  Logging changes no result."""
    lp, C = lpgen.g_grid(batch=1024, seed=2)
    prob = mp.Problem.from_lp(lp).to("cuda")
    Cd = torch.as_tensor(C, device="cuda")
    bs = mp.BatchSolver(prob, Cd)
    res = bs.solve(algorithm=alg)
    X, _ = bs.solutions()
    _, _, ro = oracle.solve_batch(lp, C, None, alg)
    diff = [b for b in range(len(res)) if res[b]["attempts"] != ro[b]["attempts"] or
            res[b]["restarts"] != ro[b]["restarts"]]
    same = [b for b in range(len(res)) if b not in set(diff)]
    assert len(diff) <= 0.25 * len(res)
    examined = 0
    for b in diff[:10] + same[:1]:
        bs.set_decision_log(att_cap=40000, chk_cap=2000, instance=b)
        r2 = bs.solve(algorithm=alg)
        att, chk = bs.decision_log()
        X2, _ = bs.solutions()
        assert np.array_equal(np.asarray(r2["attempts"]), np.asarray(res["attempts"]))   # logging is passive
        assert np.array_equal(X2, X)
        lpb = lp.with_costs(c=C[b])
        rob = oracle.solve(lpb, alg, log_capacity=40000)
        rec = compare_logs(lpb, alg, r2[b], att, chk, rob, f"C2[{b}]")
        parity_log(f"c2_decision_log[{alg},{b}]", **rec)
        examined += 1
    bs.close()
    parity_log(f"c2_divergent_instances[{alg}]", divergent=len(diff), examined=examined, total=len(res))


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


def test_step_factors_past_the_table():
    """The line-search factors of attempt j, 1 - (j+1)^-0.3 and 1 + (j+1)^-0.6 (contract step 3),
    come from a 65 536-entry table and, past it, from pow: the register kernel's logged step sizes
    obey eta_{j+1} = min(f1(j) eta_bar_j, f2(j) eta_j) on both sides of the table's end."""
    lp, C = lpgen.g_grid(batch=1, seed=2)
    # no flow can leave the source with every arc fixed at 0: a primal-infeasible grid LP that,
    # with infeasibility detection off, keeps iterating to the limit (a feasible one converges to
    # rounding and stops on 100 rejections long before 65 536 attempts)
    lp = lpgen.LP(lp.n, lp.m1, lp.m2, lp.row_ptr, lp.col_idx, lp.val, C[0], lp.q, lp.l, np.zeros(lp.n))
    bs = mp.BatchSolver(mp.Problem.from_lp(lp).to("cuda"), torch.as_tensor(C[:1], device="cuda"))
    bs.set_decision_log(att_cap=66500, chk_cap=2000, instance=0)
    r = bs.solve(algorithm="ra", iteration_limit=66100, eps_abs=0.0, eps_rel=0.0, eps_primal_infeasible=-1.0,
                 eps_dual_infeasible=-1.0)
    att, _ = bs.decision_log()
    bs.close()
    assert r[0]["attempts"] >= 66100 and len(att) >= 66000, (r[0]["status"], r[0]["attempts"])
    j = att[:-1, 0]
    f1 = 1.0 - np.power(j + 1.0, -0.3)
    f2 = 1.0 + np.power(j + 1.0, -0.6)
    want = np.minimum(f1 * att[:-1, 3], f2 * att[:-1, 2])
    np.testing.assert_allclose(att[1:, 2], want, rtol=1e-13)
    sel = (j >= 65520) & (j <= 65560)   # across the table's end
    assert sel.sum() >= 40
    np.testing.assert_allclose(att[1:, 2][sel], want[sel], rtol=1e-14)


# ---- the sharded engines (row and column shards, reading 33) ----
SHARDED_CASES = [("C1", lpgen.g_rand(50, 100, 10, seed=1)), ("mid", lpgen.g_rand(3000, 5000, 12, seed=3)),
                 ("wide", lpgen.g_rand(700, 9000, 30, seed=8))]


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("axis,shards", [("rows", 1), ("rows", 3), ("cols", 2)])
@pytest.mark.parametrize("name,lp", SHARDED_CASES)
def test_sharded_decision_log_matches_oracle(alg, axis, shards, name, lp):
    """The sharded engine's decisions (taken redundantly on every shard from the reduced partials)
    against the oracle's log, by the same criteria as the grid path's."""
    ro = oracle.solve(lp, alg, log_capacity=20000)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards, axis=axis) as s:
        s.set_decision_log(att_cap=20000, chk_cap=1000)
        rg = s.solve(algorithm=alg)
        att, chk = s.decision_log()
        # a second solve rewrites the log from its first row (the counters restart per solve)
        rg2 = s.solve(algorithm=alg)
        att2, chk2 = s.decision_log()
        assert rg2["attempts"] == rg["attempts"]
        assert np.array_equal(att, att2) and np.array_equal(chk, chk2)
    assert len(att) == rg["attempts"] and len(chk) >= 1
    parity_log(f"decision_log_sharded[{name},{alg},{axis}{shards}]",
               **compare_logs(lp, alg, rg, att, chk, ro, f"{name}/{axis}{shards}"))


def test_sharded_decision_log_skips_polishing():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=2) as s:
        s.set_decision_log(att_cap=20000, chk_cap=1000)
        r = s.solve(algorithm="ra", eps_abs=1e-2, eps_rel=1e-2, feasibility_polishing=1)
        att, chk = s.decision_log()
        ro = s.solve(algorithm="ra", eps_abs=1e-2, eps_rel=1e-2)
        att2, chk2 = s.decision_log()
    # the logged rows are the main solve's only: the same as a solve without polishing
    assert r["status"] == ro["status"] == mp.LP_OPTIMAL
    assert np.array_equal(att, att2) and np.array_equal(chk, chk2)
