"""Pins of the oracle's contract readings that PAPER.md names but does not quantify
(P:94-96): the raPDHG restart metric KKT_omega, the initial primal weight omega0 and
step eta0, the raPDHG restart candidate, and the r2HPDHG epoch reference.  Every
expected value is hand-derived in tests/golden/readings.json (derivation and citation
next to it); tests/test_oracle_mutations.py checks that a plausible slip in each of
these functions fails here.  CPU only."""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "readings.json")))
NO_SCALING = dict(ruiz_iters=0, pock_chambolle=0)


def arr(v):
    return np.array([float(t) for t in v])


def kkt_lp():
    g = GOLD["kkt_omega"]
    return lpgen.stack(arr(g["c"]), G=g["G"], h=arr(g["h"]), l=arr(g["l"]), u=arr(g["u"]))


# --------------------------------------------------------- KKT_omega (step 5) --

def test_kkt_omega_worked_example():
    g = GOLD["kkt_omega"]
    for om, want in zip(g["omega"], g["kkt_omega_squared"]):
        got = oracle.kkt_omega(kkt_lp(), om, arr(g["x"]), arr(g["y"]))
        assert got ** 2 == pytest.approx(want, rel=1e-15), om


def test_kkt_omega_satisfied_inequality_row():
    g = GOLD["kkt_omega_satisfied_row"]
    for om, want in zip(g["omega"], g["kkt_omega_squared"]):
        got = oracle.kkt_omega(kkt_lp(), om, arr(g["x"]), arr(g["y"]))
        assert got ** 2 == pytest.approx(want, rel=1e-15), om


def test_kkt_omega_is_the_weighted_norm_of_the_termination_terms():
    """omega -> pres^2 omega + dres^2 / omega is the only omega dependence: at omega = 1
    it is the plain l2 norm of (pres, dres, gap) of kkt_original."""
    lp = lpgen.g_rand(30, 50, 5, seed=21)
    rng = np.random.default_rng(3)
    x, y = rng.normal(size=lp.n), rng.normal(size=lp.m)
    k = oracle.kkt_original(lp, x, y)
    assert oracle.kkt_omega(lp, 1.0, x, y) == pytest.approx(np.sqrt(k["pres"] ** 2 + k["dres"] ** 2 + k["gap"] ** 2),
                                                             rel=1e-14)
    for om in (0.1, 7.0):
        want = np.sqrt(om * k["pres"] ** 2 + k["dres"] ** 2 / om + k["gap"] ** 2)
        assert oracle.kkt_omega(lp, om, x, y) == pytest.approx(want, rel=1e-14)


def test_rapdhg_first_reference_is_kkt_omega_of_z0():
    """raPDHG's reference at k = 0 is KKT_omega(z0) with omega0 (contract step 2); the
    first check's log row carries it (it is only replaced at a restart)."""
    g = GOLD["rapdhg_first_reference"]
    r = oracle.solve(kkt_lp(), "ra", iteration_limit=64, log_capacity=64, **NO_SCALING)
    ref = r["chk_log"][0, 2]
    assert (ref ** 2 - 9.0) / np.sqrt(2.0) == pytest.approx(g["ref_squared_minus_9_over_sqrt2"], rel=1e-14)
    r1 = oracle.solve(kkt_lp(), "ra", iteration_limit=1, **NO_SCALING)   # no restart at the limit
    assert r1["omega"] ** 2 == pytest.approx(g["omega0_squared"], rel=1e-15)


def test_rapdhg_reference_after_a_restart_is_the_candidate_metric():
    """Reading c.3 #12: after a raPDHG restart, ref := the restart candidate's KKT_omega,
    i.e. the metric logged at the restarting check."""
    lp = lpgen.g_rand(40, 80, 6, seed=2)
    r = oracle.solve(lp, "ra", check_frequency=8, iteration_limit=20000, log_capacity=4096)
    log = r["chk_log"]
    assert log[:, 4].sum() >= 2
    for i in range(1, len(log)):
        if log[i - 1, 4] == 1:
            assert log[i, 2] == log[i - 1, 1]
        elif log[i - 1, 5] == 0:
            assert log[i, 2] == log[i - 1, 2]


# ------------------------------------------------------ omega0, eta0 (step 2) --

@pytest.mark.parametrize("i", range(len(GOLD["initial_steps"]["cases"])))
def test_initial_weight_and_step(i):
    g = GOLD["initial_steps"]["cases"][i]
    K = np.array(g["K"], float)
    lp = lpgen.stack(arr(g["c"]), A=K, b=arr(g["q"]))
    kw = dict(ruiz_iters=g["ruiz_iters"], pock_chambolle=g["pock_chambolle"])
    rule = 1 if g.get("step_rule") == "constant" else 0
    om, et = oracle.initial_steps(lp, step_rule=rule, **kw)
    assert om ** 2 == pytest.approx(g["omega0_squared"], rel=1e-14)
    if "eta0" in g:
        assert et == pytest.approx(g["eta0"], rel=1e-12 if rule else 1e-15)
    else:
        assert et ** 2 == pytest.approx(g["eta0_squared"], rel=1e-14)
    # the solve starts from the same pair: the first attempt uses eta0, and with one
    # iteration (no restart at the limit) omega is still omega0
    r = oracle.solve(lp, "ra", iteration_limit=1, log_capacity=8, step_rule=rule, **kw)
    assert r["att_log"][0, 2] == et
    assert r["omega"] == om


# -------------------------------------------- raPDHG restart candidate (step 5) --

def test_restart_thresholds_are_strict_at_their_constants():
    """Reading c.3 #12's constants: just above 0.2 ref (with no rising metric) does not
    restart, just above 0.8 ref does not restart even when rising, k_in < 0.36 k does not."""
    assert not oracle.restart_test(5, 100, 0.21, 1.0, np.inf)
    assert oracle.restart_test(5, 100, 0.2, 1.0, np.inf)
    assert not oracle.restart_test(5, 100, 0.81, 1.0, 0.5)
    assert oracle.restart_test(5, 100, 0.8, 1.0, 0.5)
    assert not oracle.restart_test(35, 100, 0.9, 1.0, 0.95)


def test_restart_candidate_strictly_smaller_average():
    assert oracle.restart_candidate(1.0, 2.0) == "avg"
    assert oracle.restart_candidate(2.0, 1.0) == "cur"
    assert oracle.restart_candidate(1.5, 1.5) == "cur"               # a tie keeps the current point
    assert oracle.restart_candidate(0.0, 0.0) == "cur"
    assert oracle.restart_candidate(np.nextafter(1.0, 0.0), 1.0) == "avg"


# ---------------------------------------------- r2HPDHG reference (steps 4-5) --

def r2_lp():
    g = GOLD["r2_first_residual"]
    return lpgen.stack(arr(g["c"]), A=g["A"], b=arr(g["b"]), l=arr(g["l"]), u=arr(g["u"]))


def test_r2_first_fixed_point_residual_worked_example():
    g = GOLD["r2_first_residual"]
    r = oracle.solve(r2_lp(), "r2", check_frequency=1, iteration_limit=1, log_capacity=8, **NO_SCALING)
    assert r["att_log"][0, 1] == 1                                    # accepted at eta = eta_bar = 1
    k, metric, ref = r["chk_log"][0, :3]
    assert k == 1 and metric == g["r_P"] and ref == g["r_P"]


def test_r2_first_step_from_a_warm_start():
    g = GOLD["r2_first_step_warm"]
    r = oracle.solve(r2_lp(), "r2", iteration_limit=1, x0=arr(g["x0"]), y0=arr(g["y0"]), **NO_SCALING)
    assert r["status"] == oracle.ITERATION_LIMIT
    assert np.array_equal(r["x"], arr(g["x"])) and np.array_equal(r["y"], arr(g["y"]))


@pytest.mark.parametrize("seed", [1, 2])
def test_r2_reference_is_reset_at_every_epoch(seed):
    """Reading c.3 #12: ref = r_P of the epoch's first step.  With a check after every
    step, the check right after a restart (and the first) logs metric == ref; inside an
    epoch ref stays put."""
    lp = lpgen.g_rand(30, 60, 5, seed=seed)
    r = oracle.solve(lp, "r2", check_frequency=1, iteration_limit=400, log_capacity=1024)
    log = r["chk_log"]
    restarted = 0
    for i in range(len(log)):
        if log[i, 5] != 0:
            break
        if i == 0 or log[i - 1, 4] == 1:
            assert log[i, 2] == log[i, 1], i
            restarted += i > 0
        else:
            assert log[i, 2] == log[i - 1, 2], i
    assert restarted >= 3
