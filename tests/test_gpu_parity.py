"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY.md §8(c) c.5 parity budget):
  * scalings Dr, Dc bitwise equal (same correctly rounded ops, same order);
  * iterates after a fixed number K of accepted steps within 1e-9 relative;
  * status, iteration, attempt and restart counts identical wherever they are
    well-posed: the oracle's own counts must not move under 1-ulp
    perturbations of c and no logged decision may be a near-tie (margin < 1e-9);
    the contract's trajectories are chaotic on some instances;
  * final objective within 1e-6 relative, KKT residuals <= 1e-4 relative.
"""
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

ALGS = ["ra", "r2"]
MARGIN = 1e-9


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = max(np.linalg.norm(b), 1e-300)
    return np.linalg.norm(a - b) / den


def maxrel(a, b):
    """Elementwise error max |a - b| relative to max |b| (beside the l2 `rel`)."""
    a, b = np.asarray(a), np.asarray(b)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def close(a, b, tol):
    """Iterate parity: both the l2-relative and the elementwise error within tol."""
    return rel(a, b) <= tol and maxrel(a, b) <= tol


def min_margin(r):
    """Smallest relative margin of any discontinuous decision the oracle took."""
    mm = np.inf
    att = r.get("att_log")
    if att is not None and len(att):
        eta, eb = att[:, 2], att[:, 3]
        fin = np.isfinite(eb)
        if fin.any():
            mm = min(mm, np.min(np.abs(eta[fin] - eb[fin]) / np.maximum(eta[fin], 1e-300)))
    chk = r.get("chk_log")
    if chk is not None and len(chk):
        for k, metric, ref, last, rs, ps in chk:
            if ref > 0 and np.isfinite(ref):
                mm = min(mm, abs(metric - 0.2 * ref) / ref, abs(metric - 0.8 * ref) / ref)
            if np.isfinite(last) and metric > 0:
                mm = min(mm, abs(metric - last) / metric)
    return mm


def ulp_perturb(a, seed):
    """a with every entry moved by one relative ulp in a random direction."""
    s = np.random.default_rng(seed).choice([-1.0, 1.0], size=np.shape(a))
    return np.asarray(a) * (1.0 + s * 2.0 ** -52)


def perturbed(lp, seed):
    """The same LP with c and q perturbed entrywise by 1 ulp (random signs)."""
    return lp.with_costs(c=ulp_perturb(lp.c, seed), q=ulp_perturb(lp.q, seed + 100) if lp.m else lp.q)


def oracle_stability(lp, alg, **kw):
    """Sensitivity guard: run the oracle on the LP, on two entrywise 1-ulp
    perturbations of c and q, and as its FMA-contracted build (every step rounded differently,
    the way the GPU's fused multiply-adds do; reading 27).  Returns (result, counts_stable,
    drift): the counts are stable when the oracle's own status / iteration / attempt / restart
    counts do not move under these (and no logged decision is a near-tie), and `drift` is how
    far its own iterate moves (relative).  A GPU run with a different, equally valid
    summation order can only be held to identical counts when they are stable, and to
    max(1e-9, 100 drift)."""
    r = oracle.solve(lp, alg, log_capacity=1 << 16, **kw)
    stable = min_margin(r) >= MARGIN
    drift = 0.0
    r["obj_drift"] = 0.0
    for seed in (1, 2, "fma"):
        p = oracle.solve(lp, alg, fma=True, **kw) if seed == "fma" else oracle.solve(perturbed(lp, seed), alg, **kw)
        stable &= all(p[k] == r[k] for k in ("status", "iterations", "attempts", "restarts"))
        drift = max(drift, rel(p["x"], r["x"]), rel(p["y"], r["y"]) if lp.m else 0.0)
        r["obj_drift"] = max(r["obj_drift"], abs(p["primal_objective"] - r["primal_objective"]) /
                             (1 + abs(r["primal_objective"])))
    return r, bool(stable), drift


def obj_tol(ro):
    """Final-objective parity budget: 1e-6 relative, or 100x the
    oracle's own objective drift under 1-ulp input perturbations if larger."""
    return max(1e-6, 100 * ro["obj_drift"])


def gpu_solve(lp, alg, device=False, **kw):
    prob = mp.Problem.from_lp(lp)
    if device:
        prob = prob.to("cuda:0")
    with mp.Solver(prob) as s:
        r = s.solve(algorithm=alg, **kw)
        x, y, lam = s.solution()
    r.update(x=x, y=y, lam=lam)
    return r


def small_lps():
    yield "tiny", lpgen.tiny_spec()
    yield "C1", lpgen.g_rand(50, 100, 10, seed=1)
    yield "ragged", lpgen.g_rand(37, 61, 5, seed=7)
    yield "grid", lpgen.g_grid(batch=1)[0]
    yield "dense", lpgen.g_dense(30, 50, batch=1, seed=5)[0]


# ------------------------------------------------------------------ setup ----

@pytest.mark.parametrize("name,lp", list(small_lps()))
def test_scaling_bitwise(name, lp):
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        Dr, Dc = s.scaling()
    Dro, Dco = oracle.precondition(lp)
    assert np.array_equal(Dr, Dro) and np.array_equal(Dc, Dco)


@pytest.mark.parametrize("name,lp", list(small_lps()) + [("mid", lpgen.g_rand(3000, 5000, 12, seed=3))])
def test_spmv_scaled_vs_oracle(name, lp):
    s_or = oracle.scaled_problem(lp)
    rng = np.random.default_rng(0)
    v, w = rng.normal(size=lp.n), rng.normal(size=lp.m)
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        Kv, KTw = s.spmv_scaled(v, w)
    scaled = lpgen.LP(lp.n, lp.m1, lp.m2, lp.row_ptr, lp.col_idx, s_or["Kv"], lp.c, lp.q, lp.l, lp.u)
    Kv_o, KTw_o = oracle.spmv_pair(scaled, x=v, w=w)
    assert rel(Kv, Kv_o) <= 1e-14 and rel(KTw, KTw_o) <= 1e-14
    assert abs(Kv @ w - v @ KTw) <= 1e-12 * (abs(Kv @ w) + 1e-300)


def test_validation_errors():
    bad = lpgen.tiny_spec()
    bad.l = np.array([1.0, 0.0]); bad.u = np.array([0.0, 1.0])
    with pytest.raises(mp.LpError) as e:
        mp.Solver(mp.Problem.from_lp(bad))
    assert e.value.code == -4
    bad = lpgen.tiny_spec()
    bad.q = np.array([np.nan])
    with pytest.raises(mp.LpError) as e:
        mp.Solver(mp.Problem.from_lp(bad))
    assert e.value.code == -3
    bad = lpgen.tiny_spec()
    bad.col_idx = np.array([1, 0], np.int32)                    # unsorted row
    with pytest.raises(mp.LpError) as e:
        mp.Solver(mp.Problem.from_lp(bad))
    assert e.value.code == -2
    bad = lpgen.tiny_spec()
    bad.u = np.array([-np.inf, 1.0])
    with pytest.raises(mp.LpError) as e:
        mp.Solver(mp.Problem.from_lp(bad))
    assert e.value.code == -4


# ------------------------------------------------------- fixed-K parity ----

@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 2, 64, 256])
@pytest.mark.parametrize("name,lp", list(small_lps()))
def test_fixed_K_iterates(alg, K, name, lp):
    ro, stable, drift = oracle_stability(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    rg = gpu_solve(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    if not stable:
        pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation of c")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert close(rg["x"], ro["x"], tol), (rel(rg["x"], ro["x"]), maxrel(rg["x"], ro["x"]))
    if lp.m:
        assert close(rg["y"], ro["y"], tol), (rel(rg["y"], ro["y"]), maxrel(rg["y"], ro["y"]))
    assert abs(rg["primal_objective"] - ro["primal_objective"]) <= tol * (1 + abs(ro["primal_objective"]))


# --------------------------------------------------------- full solves -----

@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("name,lp", list(small_lps()))
def test_full_solve(alg, name, lp):
    ro, stable, drift = oracle_stability(lp, alg)
    rg = gpu_solve(lp, alg)
    assert rg["status"] == mp.LP_OPTIMAL and ro["status"] == oracle.OPTIMAL
    assert rg["rel_kkt"] <= 1e-4
    # self-certification on original data with the oracle's independent KKT routine
    k = oracle.kkt_original(lp, rg["x"], rg["y"])
    nq, nc = np.linalg.norm(lp.q), np.linalg.norm(lp.c)
    assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * nq)
    assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * nc)
    # x = Dc (x~) with l~ = l/Dc <= x~ <= u~ = u/Dc: in bounds up to the unscaling's rounding
    slack = 4e-16 * (1 + np.abs(np.where(np.isfinite(lp.u), lp.u, 0)) + np.abs(np.where(np.isfinite(lp.l), lp.l, 0)))
    assert np.all(rg["x"] >= lp.l - slack) and np.all(rg["x"] <= lp.u + slack) and np.all(rg["y"][: lp.m1] >= 0)
    if lp.obj_star is not None:
        assert abs(rg["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))
    # oracle parity (counts identical, objective within 1e-6) where the trajectory is well-posed
    if not stable or drift > 1e-6:
        pytest.skip("not well-posed: the oracle's own counts or final point move under a 1-ulp perturbation "
                    "of c, q or FMA contraction (checked above: OPTIMAL, self-certified, at the known optimum)")
    for key in ("iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    # the objective, not x: a full solve stops anywhere in a 1e-4 neighbourhood of a possibly
    # non-unique optimal face (reading 26); iterates are compared in the fixed-K tests
    assert abs(rg["primal_objective"] - ro["primal_objective"]) <= obj_tol(ro) * (1 + abs(ro["primal_objective"]))


@pytest.mark.parametrize("alg", ALGS)
def test_tiny_tight_tolerance_and_warm_start(alg):
    lp = lpgen.tiny_spec()
    rg = gpu_solve(lp, alg, eps_abs=1e-8, eps_rel=1e-8)
    assert rg["status"] == mp.LP_OPTIMAL and abs(rg["primal_objective"] - 1.0) <= 1e-6
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        r = s.solve(np.array([0.0, 1.0]), np.array([1.0]), algorithm=alg)
    assert r["status"] == mp.LP_OPTIMAL and r["iterations"] == 64


@pytest.mark.parametrize("alg", ALGS)
def test_warm_start_parity(alg):
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    rng = np.random.default_rng(3)
    x0, y0 = rng.normal(size=lp.n), rng.normal(size=lp.m)
    ro, stable, drift = oracle_stability(lp, alg, x0=x0, y0=y0, iteration_limit=128, eps_abs=0, eps_rel=0)
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        rg = s.solve(x0, y0, algorithm=alg, iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
        x, y, _ = s.solution()
    if not stable:
        pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation")
    tol = max(1e-9, 100 * drift)
    assert rg["attempts"] == ro["attempts"] and rg["restarts"] == ro["restarts"]
    assert close(x, ro["x"], tol), (rel(x, ro["x"]), maxrel(x, ro["x"]), drift)
    assert close(y, ro["y"], tol), (rel(y, ro["y"]), maxrel(y, ro["y"]), drift)


@pytest.mark.parametrize("alg", ALGS)
def test_degenerate_cases(alg):
    lp0 = lpgen.stack([1.0, -2.0, 0.5], l=[-1, -1, 0], u=[1, 3, 2])        # no rows
    rg = gpu_solve(lp0, alg, eps_abs=1e-9, eps_rel=1e-9)
    assert rg["status"] == mp.LP_OPTIMAL and np.allclose(rg["x"], [-1, 3, 0], atol=1e-8)
    lpz = lpgen.stack([1.0, 1.0], G=[[1.0, 0.0], [0.0, 0.0]], h=[1.0, -1.0], l=[0, 0], u=[5, 5])
    ro = oracle.solve(lpz, alg, eps_abs=1e-9, eps_rel=1e-9)
    rg = gpu_solve(lpz, alg, eps_abs=1e-9, eps_rel=1e-9)
    assert rg["status"] == mp.LP_OPTIMAL and rg["iterations"] == ro["iterations"]
    assert abs(rg["primal_objective"] - 1.0) <= 1e-7
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    rg = gpu_solve(lp, alg, eps_abs=1e-12, eps_rel=1e-12, iteration_limit=100)
    assert rg["status"] == mp.LP_ITERATION_LIMIT and rg["iterations"] == 100


def test_device_memory_path_equals_host_path():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    a = gpu_solve(lp, "r2")
    b = gpu_solve(lp, "r2", device=True)
    assert np.array_equal(a["x"], b["x"]) and a["attempts"] == b["attempts"]


# ------------------------------------------------------------- batches -----

def batch_drift(lp, C, alg, ro, X, Q=None, seeds=(1, 2, 3), Y=None, **kw):
    """Per-instance sensitivity of the oracle's batch solve under entrywise 1-ulp
    perturbations of C (and Q when given) and under FMA contraction (the oracle's contracted
    build, see oracle_stability): (counts stable?, iterate drift, objective drift).  The
    iterate drift is over x, and over y too when the oracle's Y is given."""
    keys = ("status", "iterations", "attempts", "restarts")
    B = C.shape[0]
    stable = np.ones(B, bool)
    dx = np.zeros(B)
    dobj = np.zeros(B)
    for seed in tuple(seeds) + ("fma",):
        if seed == "fma":
            Xp, Yp, rp = oracle.solve_batch(lp, C, Q, alg, fma=True, **kw)
        else:
            Qp = None if Q is None else ulp_perturb(Q, seed + 100)
            Xp, Yp, rp = oracle.solve_batch(lp, ulp_perturb(C, seed), Qp, alg, **kw)
        for b in range(B):
            stable[b] &= all(rp[b][k] == ro[b][k] for k in keys)
            dx[b] = max(dx[b], rel(Xp[b], X[b]), rel(Yp[b], Y[b]) if Y is not None and Y.shape[1] else 0.0)
            dobj[b] = max(dobj[b], abs(rp[b]["primal_objective"] - ro[b]["primal_objective"]) /
                          (1 + abs(ro[b]["primal_objective"])))
    return stable, dx, dobj


@pytest.mark.parametrize("alg", ALGS)
def test_grid_batch_c2_fixed_K(alg):
    """C2 batch after one check interval (K = 64 accepted steps), before the
    contract's long-run chaos sets in: every instance whose oracle counts are
    stable under 1-ulp perturbations must match counts and iterates."""
    lp, C = lpgen.g_grid(batch=1024)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    # eps = 1e-13, not 0: grid LPs often land exactly on a vertex, where an eps = 0 test is a knife edge
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=64)
    res = bs.solve(algorithm=alg, **kw)
    X, Y = bs.solutions()
    bs.close()
    Xo, Yo, ro = oracle.solve_batch(lp, C, None, alg, **kw)
    stable, dx, _ = batch_drift(lp, C, alg, ro, Xo, Y=Yo, **kw)
    assert stable.sum() >= 0.9 * 1024, stable.sum()
    parity_log(f"c2_fixed_K[{alg}]", compared=stable.sum(), total=1024)
    for b in np.nonzero(stable)[0]:
        for k in ("status", "iterations", "attempts", "restarts"):
            assert res[b][k] == ro[b][k], (b, k, res[b][k], ro[b][k])
        tol = max(1e-9, 100 * dx[b])
        assert close(X[b], Xo[b], tol), (b, rel(X[b], Xo[b]), maxrel(X[b], Xo[b]), dx[b])
        assert close(Y[b], Yo[b], max(tol, 1e-8)), (b, rel(Y[b], Yo[b]), maxrel(Y[b], Yo[b]))


@pytest.mark.parametrize("alg", ALGS)
def test_grid_batch_c2(alg):
    """C2: 1024 PyEPO-style 5x5 shortest-path LPs sharing K, full
    solves to 1e-4.  Long trajectories of this contract are chaotic (1-ulp input
    changes move the oracle's own counts on ~2% (ra) / ~14% (r2) of instances), so
    full-solve count identity is only checked loosely; every instance must be
    OPTIMAL, self-certified and at the DP optimum, and instances with identical
    counts must agree on the objective (1e-6, or 100x the oracle's own drift).
    Instances whose counts are unstable, or differ, are counted and reported, not compared."""
    lp, C = lpgen.g_grid(batch=1024)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    res = bs.solve(algorithm=alg)
    X, Y = bs.solutions()
    bs.close()
    Xo, Yo, ro = oracle.solve_batch(lp, C, None, alg)
    stable, dz, dobj = batch_drift(lp, C, alg, ro, Xo, Y=Yo)
    keys = ("status", "iterations", "attempts", "restarts")
    same = np.array([all(res[b][k] == ro[b][k] for k in keys) for b in range(1024)])
    assert same.sum() >= (0.9 if alg == "ra" else 0.6) * 1024, same.sum()
    # well-posed final point: the oracle's own (x, y) stays within 1e-6 under its perturbations;
    # elsewhere rounding is amplified along the trajectory (scripts/trace_divergence.py shows the
    # GPU-oracle and FMA-oracle distances growing alike, 1e-12 -> 1e-3) and only correctness applies
    well = stable & (dz <= 1e-6)
    compared = same & well
    parity_log(f"c2_full[{alg}]", compared=compared.sum(), same_counts=same.sum(), stable=stable.sum(),
               well_posed=well.sum(), total=1024)
    assert (well & ~same).sum() <= max(2, well.sum() // 100), (well & ~same).sum()   # guard misses, counted
    assert compared.sum() >= (0.8 if alg == "ra" else 0.4) * 1024, compared.sum()
    for b in range(1024):
        assert res[b]["status"] == mp.LP_OPTIMAL
        assert res[b]["rel_kkt"] <= 1e-4
        dp = lpgen.grid_dp_optimum(5, C[b])
        assert abs(res[b]["primal_objective"] - dp) <= 1e-3 * (1 + dp)
        if compared[b]:
            tol = max(1e-6, 100 * dobj[b])
            # objective only: grid LPs are degenerate, the 1e-4 point moves along the optimal face (reading 26)
            assert abs(res[b]["primal_objective"] - ro[b]["primal_objective"]) <= tol * (1 + dp), (b, dobj[b])
        k = oracle.kkt_original(lp.with_costs(c=C[b]), X[b], Y[b])
        assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.q))


def test_batch_equals_single_and_determinism():
    lp, C = lpgen.g_grid(batch=40)
    C[7] = C[3]
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    r1 = bs.solve(algorithm="r2")
    X1, Y1 = bs.solutions()
    r2 = bs.solve(algorithm="r2")
    X2, Y2 = bs.solutions()
    bs.close()
    assert np.array_equal(X1, X2) and np.array_equal(Y1, Y2)              # bitwise deterministic
    assert np.array_equal(X1[7], X1[3])                                    # identical instances
    for b in (0, 3, 39):
        r = gpu_solve(lp.with_costs(c=C[b]), "r2")
        assert np.array_equal(r["x"], X1[b]) and r["attempts"] == r1[b]["attempts"]


def test_dense_batch_per_instance_c3_sample():
    lp, C, Q, obj = lpgen.g_dense(200, 400, batch=256, seed=3)
    Cs, Qs = C[:8], Q[:8]
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), Cs, Qs)
    res = bs.solve(algorithm="r2", path=mp.PATH_INSTANCE)
    X, _ = bs.solutions()
    bs.close()
    Xo, Yo, ro = oracle.solve_batch(lp, Cs, Qs, "r2")
    stable, dz, dobj = batch_drift(lp, Cs, "r2", ro, Xo, Q=Qs, seeds=(1, 2), Y=Yo)
    stable &= dz <= 1e-6   # well-posed final point (see test_grid_batch_c2)
    keys = ("status", "iterations", "attempts", "restarts")
    compared = 0
    for b in range(8):
        assert res[b]["status"] == mp.LP_OPTIMAL and res[b]["rel_kkt"] <= 1e-4
        assert abs(res[b]["primal_objective"] - obj[b]) <= 1e-3 * (1 + abs(obj[b]))
        if stable[b]:
            # sensitivity guard: well-posed trajectories match the oracle exactly
            for k in keys:
                assert res[b][k] == ro[b][k], (b, k, res[b][k], ro[b][k])
            tol = max(1e-6, 100 * dobj[b])
            assert abs(res[b]["primal_objective"] - ro[b]["primal_objective"]) <= tol * (1 + abs(obj[b])), (b, dobj[b])
            compared += 1
    parity_log("c3_instance_path", compared=compared, total=8)
    assert compared >= 4, compared


@pytest.mark.parametrize("alg", ALGS)
def test_tiny_register_path_matches_generic_kernel(alg):
    """The register-resident warp kernel (auto path for C2-sized LPs) and the
    generic per-instance kernel implement the same arithmetic in the same order."""
    lp, C = lpgen.g_grid(batch=256, seed=11)
    out = {}
    for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
        res = bs.solve(algorithm=alg, path=path)
        X, Y = bs.solutions()
        bs.close()
        out[path] = (res, X, Y)
    (ra_, Xa, Ya), (rb_, Xb, Yb) = out[mp.PATH_AUTO], out[mp.PATH_INSTANCE]
    same = [ra_[b]["attempts"] == rb_[b]["attempts"] and ra_[b]["restarts"] == rb_[b]["restarts"]
            for b in range(256)]
    parity_log(f"tiny_vs_generic[{alg}]", same_counts=sum(same), total=256)
    assert sum(same) >= (0.9 if alg == "ra" else 0.6) * 256, sum(same)
    for b in range(256):
        assert ra_[b]["status"] == mp.LP_OPTIMAL and rb_[b]["status"] == mp.LP_OPTIMAL
        # same arithmetic (common.cuh), different summation order: identical counts -> same point
        tol = 1e-6 if same[b] else 1e-3
        assert abs(ra_[b]["primal_objective"] - rb_[b]["primal_objective"]) <= tol * (1 + abs(rb_[b]["primal_objective"]))
    # before the long-run chaos: one check interval, identical counts and iterates
    bsA = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    rA = bsA.solve(algorithm=alg, path=mp.PATH_AUTO, iteration_limit=64, eps_abs=0.0, eps_rel=0.0)
    XA, _ = bsA.solutions()
    bsA.close()
    bsB = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    rB = bsB.solve(algorithm=alg, path=mp.PATH_INSTANCE, iteration_limit=64, eps_abs=0.0, eps_rel=0.0)
    XB, _ = bsB.solutions()
    bsB.close()
    agree = sum(rA[b]["attempts"] == rB[b]["attempts"] and rel(XA[b], XB[b]) <= 1e-9 for b in range(256))
    assert agree >= 0.95 * 256, agree


@pytest.mark.parametrize("engine,expect", [("single", 4), ("dmma", 32), ("sharded", 4)])
def test_verbose_lines(engine, expect):
    """verbose = 1: one device printf line per display_frequency-th check of every
    instance, on every engine; off by default."""
    import subprocess
    import sys
    mk = {"single": "mp.Solver(mp.Problem.from_lp(lpgen.g_rand(50, 100, 10, seed=1)))",
          "dmma": "mp.BatchSolver(mp.Problem.from_lp(d[0]), d[1], d[2])",
          "sharded": "mp.ShardedSolver(mp.Problem.from_lp(lpgen.g_rand(50, 100, 10, seed=1)), virtual_shards=2)"}[engine]
    path = ", path=mp.PATH_DMMA" if engine == "dmma" else ""
    code = ("import lpgen, paper_2412_09734_b200 as mp\n"
            "d = lpgen.g_dense(60, 90, batch=8, seed=5)\n"
            "for v in (0, 1):\n"
            f"    s = {mk}\n"
            f"    s.solve(algorithm='ra', verbose=v, display_frequency=1, iteration_limit=256, eps_abs=0.0, eps_rel=0.0{path})\n"
            "    s.close()\n"
            "    print('END', v, flush=True)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__))).stdout
    first, second = out.split("END 0")
    assert "[mpax]" not in first
    lines = [l for l in second.splitlines() if l.startswith("[mpax]")]
    assert len(lines) == expect and "iter      256" in lines[-1], out
