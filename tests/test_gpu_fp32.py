"""GPU parity of the fp32-storage grid path (lp_options.precision = LP_FP32; SURVEY §8(f) row 4,
P:286-295, reading 39) against the fp32 build of the oracle, through the C ABI.

The two programs round differently by design -- the oracle is the all-single program MPAX runs by
default, the GPU path stores K~ and the iterates in fp32 but computes every element and every
reduction in fp64 -- so counts and iterates are compared within the fp32 rounding amplitude that
the oracle itself exhibits: `dev` = distance between the fp32 and the fp64 oracle on the same LP
and K.  Full solves are compared by outcome (status, self-certified KKT, objective) and by
iteration counts within a band."""
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
from tests.test_gpu_grid import CASES, grid_solve  # noqa: E402
from tests.test_gpu_parity import rel  # noqa: E402

ALGS = ["ra", "r2"]


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 2, 8])
@pytest.mark.parametrize("name,lp", CASES)
def test_fp32_fixed_K(alg, K, name, lp):
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    o64 = oracle.solve(lp, alg, **kw)
    o32 = oracle.solve(lp, alg, precision="fp32", **kw)
    g32 = grid_solve(lp, alg, precision="fp32", **kw)
    g64 = grid_solve(lp, alg, **kw)
    dev = rel(o32["x"], o64["x"])
    assert g32["status"] == o32["status"] == mp.LP_ITERATION_LIMIT
    assert g32["iterations"] == o32["iterations"] == K
    if o32["attempts"] == o64["attempts"]:   # the fp32 program takes the fp64 decisions here
        assert g32["attempts"] == o32["attempts"], (g32["attempts"], o32["attempts"])
    for v in ("x", "y", "lam"):
        if v == "y" and not lp.m:
            continue
        # the fp32 program's own distance from fp64 on this vector (its rounding amplitude here;
        # the reduced costs c - K'y / D_c carry cancellation, so each vector gets its own)
        dv = rel(o32[v], o64[v])
        tol = max(4 * dv, 2e-6)
        assert rel(g32[v], o32[v]) <= tol, (v, rel(g32[v], o32[v]), dv)
        assert rel(g32[v], o64[v]) <= tol, (v, rel(g32[v], o64[v]), dv)
    # fp32 storage is a different program from fp64: it must not silently be the fp64 path
    if dev > 0 and lp.nnz > 100:
        assert not np.array_equal(g32["x"], g64["x"])
    parity_log(f"fp32_fixed_K{K}[{name},{alg}]", compared=1, total=1, dev=dev, gpu_vs_oracle32=rel(g32["x"], o32["x"]))


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("name,lp", CASES)
def test_fp32_full_solve(alg, name, lp):
    o32 = oracle.solve(lp, alg, precision="fp32")
    g32 = grid_solve(lp, alg, precision="fp32")
    assert o32["status"] == mp.LP_OPTIMAL
    assert g32["status"] == mp.LP_OPTIMAL and g32["rel_kkt"] <= 1e-4
    # self-certified in fp64 on the returned (x, y): the termination test of P:96 holds
    k = oracle.kkt_original(lp, g32["x"], g32["y"])
    assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.q))
    assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.c))
    assert k["gap"] <= (1 + 1e-6) * (1e-4 + 1e-4 * (abs(k["pobj"]) + abs(k["dobj"])))
    if lp.obj_star is not None:
        assert abs(g32["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))
    # two 1e-4-accurate solutions of the same LP: objectives within 1e-3 relative
    assert abs(g32["primal_objective"] - o32["primal_objective"]) <= 1e-3 * (1 + abs(o32["primal_objective"]))
    # the same method: accepted-step counts within a band around the fp32 program's
    assert 0.5 * o32["iterations"] - 64 <= g32["iterations"] <= 2 * o32["iterations"] + 64, \
        (g32["iterations"], o32["iterations"])
    parity_log(f"fp32_full[{name},{alg}]", compared=1, total=1, gpu_iters=g32["iterations"],
               oracle32_iters=o32["iterations"])


def test_fp32_split_matches_unsplit(monkeypatch):
    """The two-pass phase B (column halves of K~, fp32 copies of both halves) against the
    one-pass sweep: same method, summation order differs only in the split."""
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    kw = dict(eps_abs=0.0, eps_rel=0.0, iteration_limit=8, precision="fp32")
    a = grid_solve(lp, "ra", **kw)
    monkeypatch.setenv("MPAX_GRID_SPLIT", "1")
    b = grid_solve(lp, "ra", **kw)
    assert a["attempts"] == b["attempts"]
    assert rel(b["x"], a["x"]) <= 1e-6 and rel(b["y"], a["y"]) <= 1e-6


def test_fp32_refused_off_the_grid_path():
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        with pytest.raises(mp.LpError) as e:
            s.solve(algorithm="r2", path=mp.PATH_INSTANCE, precision="fp32")
        assert e.value.code == -10
        r = s.solve(algorithm="r2", path=mp.PATH_GRID, precision="fp32")
        assert r["status"] == mp.LP_OPTIMAL


def test_fp32_deterministic():
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    a = grid_solve(lp, "r2", precision="fp32", iteration_limit=300, eps_abs=0.0, eps_rel=0.0)
    b = grid_solve(lp, "r2", precision="fp32", iteration_limit=300, eps_abs=0.0, eps_rel=0.0)
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"]) and a["attempts"] == b["attempts"]


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("kind", ["primal", "dual"])
def test_fp32_infeasibility_certificates(kind, alg):
    """fp32 storage with infeasibility detection (reading 35) at tolerances a single-precision
    ray can meet (1e-5: the default 1e-8 lies below fp32's rounding of a unit ray).  A ray is the
    difference of two nearly equal fp32 points, so whether it meets the tolerance within the
    limit depends on the trajectory's rounding: the GPU must certify at least as many of the
    four planted LPs as the fp32 oracle less one, never the wrong kind, and every GPU certificate
    must be a Farkas certificate of the fp64 problem to the fp32 level (1e-4)."""
    from tests.test_oracle_infeasibility import farkas_dual_ok, farkas_primal_ok
    want = mp.LP_PRIMAL_INFEASIBLE if kind == "primal" else mp.LP_DUAL_INFEASIBLE
    certified = certified_o = 0
    for seed in range(4):
        lp = lpgen.g_infeasible(kind, seed)
        tol = dict(eps_primal_infeasible=1e-5, eps_dual_infeasible=1e-5)
        o32 = oracle.solve(lp, alg, iteration_limit=10000, precision="fp32", **tol)
        with mp.Solver(mp.Problem.from_lp(lp)) as s:
            r = s.solve(algorithm=alg, path=mp.PATH_GRID, precision="fp32", iteration_limit=10000, **tol)
            x, y, _ = s.solution()
        assert r["status"] in (want, mp.LP_ITERATION_LIMIT, mp.LP_NUMERICAL_ERROR), (seed, r["status"])
        certified_o += o32["status"] == want
        if r["status"] == want:
            certified += 1
            # unit rays to the fp32 level (the norm is taken before the stored iterate rounds)
            if want == mp.LP_PRIMAL_INFEASIBLE:
                assert abs(np.linalg.norm(y) - 1) <= 1e-6 and farkas_primal_ok(lp, y, tol=1e-4)
            else:
                assert abs(np.linalg.norm(x) - 1) <= 1e-6 and farkas_dual_ok(lp, x, tol=1e-4)
    assert certified >= max(1, certified_o - 1), (certified, certified_o)
    parity_log(f"fp32_infeasibility[{kind},{alg}]", certified=certified, oracle32_certified=certified_o, total=4)


@pytest.mark.parametrize("alg", ALGS)
def test_fp32_polishing_and_warm_start(alg):
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        r = s.solve(algorithm=alg, path=mp.PATH_GRID, precision="fp32", eps_abs=1e-3, eps_rel=1e-3,
                    feasibility_polishing=1)
        x, y, lam = s.solution()
        assert r["status"] == mp.LP_OPTIMAL and r["polish"] in (1, 2)
        k = oracle.kkt_original(lp, x, y)
        if r["polish"] == 1:   # the polished residuals, recomputed in fp64 on the returned point
            assert k["pres"] <= 1.05 * 1e-6 * (1 + np.linalg.norm(lp.q))
            assert k["dres"] <= 1.05 * 1e-6 * (1 + np.linalg.norm(lp.c))
        # warm start from the (unpolished) fp32 solution: no more accepted steps to 1e-4 than cold
        cold = s.solve(algorithm=alg, path=mp.PATH_GRID, precision="fp32")
        xc, yc, _ = s.solution()
        warm = s.solve(xc, yc, algorithm=alg, path=mp.PATH_GRID, precision="fp32")
        assert warm["status"] == cold["status"] == mp.LP_OPTIMAL
        assert warm["iterations"] <= cold["iterations"]
