"""Pins of the CPU oracle (oracle/mpax_oracle.c) to things other than itself:
SPEC.md's hand-derived worked examples (tests/golden/spec_examples.json, each
cited), closed forms, invariants and special cases.
CPU only."""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def arr(v):
    return np.array([float(t) if not isinstance(t, str) else float(t.replace("inf", "inf")) for t in v])


def lp_from(d, c=None):
    G = np.array(d["G"], float)
    return lpgen.stack(arr(d["c"]) if c is None else c, G=G, h=arr(d["h"]), l=arr(d["l"]), u=arr(d["u"]))


# ----------------------------------------------------------------- Step 0/1 --

def test_stacking_spec_s45():
    g = GOLD["stacking"]
    lp = lpgen.stack([0.0], G=g["G"], h=g["h"], A=g["A"], b=g["b"])
    assert np.array_equal(lp.dense_K(), np.array(g["K"], float))
    assert np.array_equal(lp.q, arr(g["q"])) and lp.m1 == g["m1"]
    lp0 = lpgen.stack([0.0], A=g["A"], b=g["b"])          # m1 = 0 gives K = A
    assert lp0.m1 == 0 and np.array_equal(lp0.dense_K(), np.array(g["A"], float))


def test_validation_spec_s55_57():
    ok = lpgen.tiny_spec()
    assert oracle.validate(ok) == 0
    bad = lpgen.tiny_spec()
    bad.l = np.array([1.0, 0.0]); bad.u = np.array([0.0, 1.0])
    assert oracle.validate(bad) == -4                          # crossed bounds
    bad = lpgen.tiny_spec()
    bad.c = np.array([np.nan, 1.0])
    assert oracle.validate(bad) == -3
    bad = lpgen.tiny_spec()
    bad.row_ptr = np.array([0, 1], np.int64)                   # row_ptr[m] != nnz
    assert oracle.validate(bad) == -2
    with pytest.raises(ValueError):                            # rhs length mismatch
        lpgen.stack([1.0], A=[[1.0]], b=[1.0, 2.0])


def test_ruiz_one_round_spec_s201():
    g = GOLD["ruiz_one_round"]
    lp = lpgen.stack([1.0, 1.0], A=g["K"], b=[0.0, 0.0])
    s = oracle.scaled_problem(lp, ruiz_iters=1, pock_chambolle=0)
    assert np.array_equal(s["Dr"], arr(g["row_scale"]))
    assert np.array_equal(s["Dc"], arr(g["col_scale"]))
    K = np.zeros((2, 2)); rows = np.repeat(np.arange(2), np.diff(lp.row_ptr)); K[rows, lp.col_idx] = s["Kv"]
    assert np.array_equal(K, np.array(g["K_scaled"], float))


def test_ruiz_fixed_point_spec_s202():
    g = GOLD["ruiz_fixed_point"]
    lp = lpgen.stack([1.0, 1.0], A=g["K"], b=[0.0, 0.0])
    s = oracle.scaled_problem(lp, ruiz_iters=10, pock_chambolle=0)
    assert np.array_equal(s["Dr"], arr(g["row_scale"])) and np.array_equal(s["Dc"], arr(g["col_scale"]))


@pytest.mark.parametrize("seed", range(20))
def test_ruiz_equilibrates_spec_s628(seed):
    """Acceptance #5: after 10 Ruiz rounds every nonzero row/column inf-norm of
    a random 5%-dense matrix lies in [0.9, 1.1]."""
    rng = np.random.default_rng(1000 + seed)
    K = np.where(rng.uniform(size=(60, 40)) < 0.05, rng.normal(size=(60, 40)) * 10 ** rng.uniform(-3, 3, size=(60, 40)), 0.0)
    lp = lpgen.stack(np.ones(40), A=K, b=np.zeros(60))
    s = oracle.scaled_problem(lp, ruiz_iters=10, pock_chambolle=0)
    Ks = np.zeros_like(K); rows = np.repeat(np.arange(60), np.diff(lp.row_ptr)); Ks[rows, lp.col_idx] = s["Kv"]
    rn, cn = np.abs(Ks).max(axis=1), np.abs(Ks).max(axis=0)
    assert np.all((rn[rn > 0] >= 0.9) & (rn[rn > 0] <= 1.1))
    assert np.all((cn[cn > 0] >= 0.9) & (cn[cn > 0] <= 1.1))


def test_pock_chambolle_spec_s211_213():
    g = GOLD["pock_chambolle_scalar"]
    lp = lpgen.stack([1.0], A=g["K"], b=[1.0])
    s = oracle.scaled_problem(lp, ruiz_iters=0, pock_chambolle=1)
    assert s["Kv"][0] == pytest.approx(1.0, rel=0, abs=4.5e-16)  # 2 (1/sqrt2)^2 rounds to 1 - 2^-52
    # a zero row keeps scale 1 and stays zero
    lp = lpgen.stack([1.0, 1.0], A=[[2.0, 1.0], [0.0, 0.0]], b=[1.0, 0.0])
    s = oracle.scaled_problem(lp, ruiz_iters=0, pock_chambolle=1)
    assert s["Dr"][1] == 1.0
    # closed form of PC alpha=1 on [[2,1]]: rho = 3, gamma = (2, 1)
    assert s["Dr"][0] == pytest.approx(1 / np.sqrt(3), rel=1e-15)
    assert np.allclose(s["Dc"], [1 / np.sqrt(2), 1.0], rtol=1e-15)
    # magnitude only
    a = oracle.scaled_problem(lpgen.stack([1, 1.0], A=[[2.0, -1.0], [-3.0, 4.0]], b=[0, 0.0]))
    b = oracle.scaled_problem(lpgen.stack([1, 1.0], A=[[2.0, 1.0], [3.0, 4.0]], b=[0, 0.0]))
    assert np.array_equal(a["Dr"], b["Dr"]) and np.array_equal(a["Dc"], b["Dc"])


def test_scaling_invariants_spec_s222_s227():
    lp = lpgen.g_rand(40, 80, 6, seed=11)
    s = oracle.scaled_problem(lp)
    assert np.all(np.sign(s["Kv"]) == np.sign(lp.val))            # sign and pattern kept
    assert np.all(s["Dr"] > 0) and np.all(s["Dc"] > 0)
    # K~ = Dr K Dc (definition), and c~, q~, l~, u~ (contract step 1)
    rows = np.repeat(np.arange(lp.m), np.diff(lp.row_ptr))
    assert np.allclose(s["Kv"], lp.val * s["Dr"][rows] * s["Dc"][lp.col_idx], rtol=1e-15, atol=0)
    assert np.allclose(s["c"], lp.c * s["Dc"], rtol=1e-15)
    assert np.allclose(s["q"], lp.q * s["Dr"], rtol=1e-15)
    fin = np.isfinite(lp.l)
    assert np.allclose(s["l"][fin], lp.l[fin] / s["Dc"][fin], rtol=1e-15)
    assert np.array_equal(np.isfinite(s["u"]), np.isfinite(lp.u))
    # unscale(scale(z)) = z to 1e-14
    x = np.random.default_rng(0).normal(size=lp.n)
    assert np.allclose((x / s["Dc"]) * s["Dc"], x, rtol=1e-14, atol=0)


def test_transpose_exact():
    import scipy.sparse as sp
    lp = lpgen.g_rand(30, 50, 5, seed=3)
    s = oracle.scaled_problem(lp)
    K = sp.csr_matrix((s["Kv"], lp.col_idx.astype(np.int64), lp.row_ptr), shape=(lp.m, lp.n))
    KT = K.T.tocsr(); KT.sort_indices()
    assert np.array_equal(KT.indptr, s["KT_row_ptr"])
    assert np.array_equal(KT.indices, s["KT_col_idx"])
    assert np.array_equal(KT.data, s["KTv"])


# ------------------------------------------------------------- linear algebra --

def test_spmv_pair_examples_and_adjoint_s134_s159():
    I3 = lpgen.stack(np.zeros(3), A=np.eye(3), b=np.zeros(3))
    Kx, _ = oracle.spmv_pair(I3, x=[1, 2, 3])
    assert np.array_equal(Kx, [1, 2, 3])
    M = lpgen.stack(np.zeros(2), A=[[1, 2], [3, 4]], b=np.zeros(2))
    Kx, KTw = oracle.spmv_pair(M, x=[1, 1], w=[1, 1])
    assert np.array_equal(Kx, [3, 7]) and np.array_equal(KTw, [4, 6])
    lp = lpgen.g_rand(200, 300, 7, seed=5)
    rng = np.random.default_rng(1)
    v, w = rng.normal(size=lp.n), rng.normal(size=lp.m)
    Kv, KTw = oracle.spmv_pair(lp, x=v, w=w)
    assert abs(Kv @ w - v @ KTw) <= 1e-10 * abs(Kv @ w)
    Kd = lp.dense_K()                                             # dense library product
    assert np.max(np.abs(Kv - Kd @ v)) <= 1e-12 * np.max(np.abs(Kd @ v))
    assert np.max(np.abs(KTw - Kd.T @ w)) <= 1e-12 * np.max(np.abs(Kd.T @ w))


# ------------------------------------------------------------------- Step 3 --

def test_projections_s273_285():
    g = GOLD["project_box"]
    assert np.array_equal(oracle.project_box(arr(g["x"]), arr(g["l"]), arr(g["u"])), arr(g["out"]))
    g = GOLD["project_box_free"]
    assert np.array_equal(oracle.project_box(arr(g["x"]), arr(g["l"]), arr(g["u"])), arr(g["out"]))
    g = GOLD["project_dual"]
    assert np.array_equal(oracle.project_dual(arr(g["y"]), g["m1"]), arr(g["out"]))
    assert np.array_equal(oracle.project_dual([-1.0, 2.0], 0), [-1.0, 2.0])     # m1 = 0 identity
    x = np.array([0.3, -0.2])
    assert np.array_equal(oracle.project_box(x, [-1, -1], [1, 1]), x)           # idempotence


def test_pdhg_step_s293_295():
    g = GOLD["pdhg_fixed_point"]
    lp = lp_from(g)
    for tau, sigma in [(0.5, 0.5), (3.0, 0.1), (1e-3, 7.0)]:
        xo, yo = oracle.pdhg_step(lp, arr(g["x"]), arr(g["y"]), tau, sigma)
        assert np.array_equal(xo, arr(g["out_x"])) and np.array_equal(yo, arr(g["out_y"]))
    g = GOLD["pdhg_step"]
    xo, yo = oracle.pdhg_step(lp_from(g), arr(g["x"]), arr(g["y"]), g["tau"], g["sigma"])
    assert np.array_equal(xo, arr(g["out_x"])) and np.array_equal(yo, arr(g["out_y"]))
    # K = 0 decouples into projected gradient steps on c'x and -q'y
    lp = lpgen.stack([1.0, -2.0], A=np.zeros((1, 2)), b=[3.0], l=[-5, -5], u=[5, 5])
    xo, yo = oracle.pdhg_step(lp, [0.0, 0.0], [1.0], 0.5, 0.25)
    assert np.array_equal(xo, [-0.5, 1.0]) and np.array_equal(yo, [1.75])


def test_line_search_s323_325():
    g = GOLD["line_search"]
    eb, acc, _ = oracle.step_size(g["rejected_eta"], g["omega"], g["dx2"], g["dy2"], g["interaction"], 1)
    assert eb == g["eta_bar"] and not acc
    eb, acc, _ = oracle.step_size(g["accepted_eta"], g["omega"], g["dx2"], g["dy2"], g["interaction"], 1)
    assert eb == g["eta_bar"] and acc
    # interaction = 0: always accept, eta grows by (1 + (j+1)^-0.6)
    for j in (1, 7, 100):
        eb, acc, en = oracle.step_size(0.3, 2.0, 1.0, 4.0, 0.0, j)
        assert eb == np.inf and acc and en == pytest.approx(0.3 * (1 + (j + 1) ** -0.6), rel=1e-15)
    # next eta = min((1-(j+1)^-0.3) eta_bar, (1+(j+1)^-0.6) eta): closed form
    eb, acc, en = oracle.step_size(10.0, 1.0, 1.0, 1.0, 1.0, 3)
    assert en == pytest.approx(min((1 - 4 ** -0.3) * 1.0, (1 + 4 ** -0.6) * 10.0), rel=1e-15)
    # accepted steps satisfy 2 eta |I| <= M, so r_P^2 = M/eta - 2I >= 0 (SURVEY c.4)
    rng = np.random.default_rng(7)
    for _ in range(2000):
        eta, om = 10 ** rng.uniform(-3, 1), 10 ** rng.uniform(-2, 2)
        dx2, dy2, I = rng.exponential(), rng.exponential(), rng.normal()
        eb, acc, _ = oracle.step_size(eta, om, dx2, dy2, I, 5)
        if acc:
            assert (om * dx2 + dy2 / om) / eta - 2 * I >= -1e-12 * (om * dx2 + dy2 / om) / eta


def test_halpern_s303_305():
    g = GOLD["halpern"]
    assert np.array_equal(oracle.halpern(g["k"], arr(g["z"]), arr(g["w"]), arr(g["z0"])), arr(g["out"]))
    rng = np.random.default_rng(2)
    z, w, z0 = rng.normal(size=(3, 5))
    assert np.allclose(oracle.halpern(0, z0, w, z0), w, rtol=0, atol=1e-15)  # k=0, z=z0: z1 = PDHG(z0)
    for k in (0, 3, 50):
        assert np.allclose(oracle.halpern(k, z0, z0, z0), z0, rtol=1e-15)    # fixed point
    # affine with coefficients summing to 1: translation equivariance
    t = 3.7
    assert np.allclose(oracle.halpern(4, z + t, w + t, z0 + t), oracle.halpern(4, z, w, z0) + t, atol=1e-14)


def test_average_s313_315():
    g = GOLD["average"]
    avg, W = np.zeros(1), 0.0
    for p, wt in zip(g["points"], g["weights"]):
        avg, W = oracle.average_update(avg, p, W, wt)
    assert np.array_equal(avg, arr(g["out"])) and W == 4.0
    avg, W = oracle.average_update([123.0], [5.0], 0.0, 0.7)                 # single point
    assert np.array_equal(avg, [5.0])


def test_primal_weight_s333_335():
    g = GOLD["primal_weight"]
    assert oracle.primal_weight(g["omega"], g["dx"], g["dy"]) == g["out"]
    assert oracle.primal_weight(3.0, 0.0, 1.0) == 3.0
    assert oracle.primal_weight(3.0, 1.0, 0.0) == 3.0
    assert oracle.primal_weight(2.0, 1.0, 8.0) == 4.0                        # sqrt(2 * 8)


# ------------------------------------------------------------------- Step 5 --

def test_kkt_s395_397():
    g = GOLD["kkt_at_optimum"]
    lp = lp_from(g)
    k = oracle.kkt_original(lp, arr(g["x"]), arr(g["y"]))
    for key in ("pres", "dres", "pobj", "dobj", "gap"):
        assert k[key] == g[key], key
    g2 = GOLD["kkt_infeasible_point"]
    assert oracle.kkt_original(lp, arr(g2["x"]), arr(g2["y"]))["pres"] == g2["pres"]
    k = oracle.kkt_original(lp_from(g, c=np.zeros(2)), arr(g["x"]), [0.0])
    assert k["dres"] == 0 and k["dobj"] == 0


def test_kkt_bound_terms_closed_form():
    """Hand-checked cases that exercise every term of the dual objective and
    dual residual (contract step 5): finite l, finite u, free columns."""
    lp = lpgen.stack([1.0], l=[2.0], u=[5.0])            # min x on [2,5]: x=2, lambda=1
    k = oracle.kkt_original(lp, [2.0], [])
    assert (k["pobj"], k["dobj"], k["gap"], k["dres"]) == (2.0, 2.0, 0.0, 0.0)
    lp = lpgen.stack([-1.0], l=[2.0], u=[5.0])           # min -x: x=5, lambda=-1
    k = oracle.kkt_original(lp, [5.0], [])
    assert (k["pobj"], k["dobj"], k["gap"], k["dres"]) == (-5.0, -5.0, 0.0, 0.0)
    lp = lpgen.stack([1.0, -3.0], l=[-np.inf, 0.0], u=[np.inf, np.inf])    # free: |lambda|; [0,inf): lambda-
    k = oracle.kkt_original(lp, [0.0, 0.0], [])
    assert k["dres"] == pytest.approx(np.sqrt(1 + 9), rel=1e-15)
    # equality row residual is signed both ways, >= row only one way
    lp = lpgen.stack([0.0], G=[[1.0]], h=[1.0], A=[[1.0]], b=[1.0])
    assert oracle.kkt_original(lp, [3.0], [0.0, 0.0])["pres"] == 2.0        # only the = row violated
    assert oracle.kkt_original(lp, [0.0], [0.0, 0.0])["pres"] == pytest.approx(np.sqrt(2), rel=1e-15)
    k = oracle.kkt_original(lp, [1.0], [2.0, -0.5])                         # dobj = q'y
    assert k["dobj"] == 1.5 and k["dres"] == pytest.approx(1.5)


def test_termination_s405_407():
    z = dict(pres=0.0, dres=0.0, pobj=0.0, dobj=0.0, gap=0.0)
    assert oracle.termination(z, 1.0, 1.0, 1e-4, 1e-4)
    big = dict(pres=0.0, dres=0.0, pobj=1.0, dobj=0.0, gap=1.0)
    assert not oracle.termination(big, 1.0, 1.0, 1e-4, 1e-4)
    # thresholds exactly met (<=): eps_abs = 0.125, eps_rel = 0 for each term
    assert oracle.termination(dict(pres=0.125, dres=0.125, pobj=1.0, dobj=1.0, gap=0.125), 0, 0, 0.125, 0.0)
    assert not oracle.termination(dict(pres=0.125000001, dres=0, pobj=1, dobj=1, gap=0), 0, 0, 0.125, 0.0)
    # each term uses its own scale: ||q||, ||c||, |pobj|+|dobj|
    assert oracle.termination(dict(pres=2.0, dres=0, pobj=0, dobj=0, gap=0), 4.0, 0.0, 0.0, 0.5)
    assert not oracle.termination(dict(pres=2.0, dres=0, pobj=0, dobj=0, gap=0), 0.0, 4.0, 0.0, 0.5)
    assert oracle.termination(dict(pres=0, dres=2.0, pobj=0, dobj=0, gap=0), 0.0, 4.0, 0.0, 0.5)
    assert oracle.termination(dict(pres=0, dres=0, pobj=3.0, dobj=-1.0, gap=2.0), 0, 0, 0.0, 0.5)
    assert oracle.rel_kkt(dict(pres=1.0, dres=4.0, pobj=1.0, dobj=1.0, gap=0.0), 1.0, 1.0) == 2.0


def test_restart_s415_417():
    g = GOLD
    assert oracle.restart_test(5, 100, g["restart_sufficient"]["metric"], 1.0, np.inf) is True
    r = g["restart_necessary_stall"]
    assert oracle.restart_test(5, 100, r["metric"], r["ref"], r["last"]) is True
    r = g["restart_none"]
    assert oracle.restart_test(5, 100, r["metric"], r["ref"], r["last"]) is False
    assert oracle.restart_test(64, 64, 1.0, 1.0, 0.5) is True        # artificial: k_in >= 0.36 k
    assert oracle.restart_test(35, 100, 1.0, 1.0, 0.5) is False
    assert oracle.restart_test(36, 100, 1.0, 1.0, 0.5) is True
    assert oracle.restart_test(5, 100, 0.2, 1.0, 0.1) is True        # boundary (<=) sufficient
    assert oracle.restart_test(5, 100, 0.8, 1.0, 0.8) is False       # not rising


# ------------------------------------------------- constant-step variant --

def test_spectral_norm_s144_146():
    """Power iteration for sigma_max: closed forms and the SVD."""
    assert oracle.spectral_norm(lpgen.stack([0, 0.0], A=[[3, 0], [0, 1]], b=[0, 0])) == pytest.approx(3.0, rel=1e-12)
    assert oracle.spectral_norm(lpgen.stack([0, 0.0], A=[[0, 1], [0, 0]], b=[0, 0])) == pytest.approx(1.0, rel=1e-12)
    rng = np.random.default_rng(4)
    for shape in [(10, 10), (25, 40), (60, 30)]:
        K = rng.normal(size=shape)
        lp = lpgen.stack(np.zeros(shape[1]), A=K, b=np.zeros(shape[0]))
        s = oracle.spectral_norm(lp, iters=2000)
        assert s == pytest.approx(np.linalg.svd(K, compute_uv=False)[0], rel=1e-8)
        assert s <= np.linalg.svd(K, compute_uv=False)[0] * (1 + 1e-12)      # never above sigma_max
    assert oracle.spectral_norm(lpgen.stack([0, 0.0], A=np.zeros((2, 2)), b=[0, 0])) == 0.0
