"""GPU parity of infeasibility detection (DESIGN.md §3
reading 35) on every solver path against the oracle: the same status on every
instance, and certificate rays that pass the Farkas check independently of
both.  With the constant step the GPU and oracle trajectories agree to ~1e-15
on these instances, so the detection iteration and the rays must match too;
with the adaptive step the iterates of an infeasible LP grow and the line
search makes them chaotic (the two trajectories are 1e-9..1e-2 apart after
256 steps, as the oracle is from its own 1-ulp perturbations), so only the
verdict and the certificate's validity are compared."""
import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from tests.test_oracle_infeasibility import farkas_dual_ok, farkas_primal_ok, spec_dual_infeasible, \
    spec_primal_infeasible  # noqa: E402

ALGS = ["ra", "r2"]
RULES = ["adaptive", "constant"]
PI, DI = mp.LP_PRIMAL_INFEASIBLE, mp.LP_DUAL_INFEASIBLE
LIMIT = 10000


def want_status(kind):
    return PI if kind == "primal" else DI


def check_rays(lp, status, x, y):
    if status == PI:
        assert abs(np.linalg.norm(y) - 1) <= 1e-12 and farkas_primal_ok(lp, y)
    elif status == DI:
        assert abs(np.linalg.norm(x) - 1) <= 1e-12 and farkas_dual_ok(lp, x)


def same_frac(rule):
    return 1.0 if rule == "constant" else 0.0


def compare(lp, res_g, X, Y, res_o, Xo, Yo, min_same=0.8):
    """min_same = 1 (constant step): statuses identical on every instance, and the
    detection iteration identical on >= min_same of them with rays equal to the
    oracle's to 1e-6.  min_same = 0 (adaptive step, chaotic): the verdicts may differ
    only by one side reaching the limit first -- the GPU must never give a status the
    oracle contradicts (a certificate of the other kind, or OPTIMAL vs a certificate).
    Every GPU ray is checked against the Farkas alternative."""
    same = 0
    undecided = (oracle.ITERATION_LIMIT, oracle.NUMERICAL_ERROR)
    for b in range(len(res_o)):
        sg, so = int(res_g[b]["status"]), int(res_o[b]["status"])
        if min_same > 0:
            assert sg == so or (so in undecided and sg in undecided), (b, sg, so)
        else:
            assert sg == so or sg in undecided or so in undecided, (b, sg, so)
        check_rays(lp, sg, X[b], Y[b])
        if res_g[b]["iterations"] == res_o[b]["iterations"]:
            same += 1
            if sg in (PI, DI) and sg == so:
                ray_g, ray_o = (Y[b], Yo[b]) if sg == PI else (X[b], Xo[b])
                if min_same > 0:
                    assert np.linalg.norm(ray_g - ray_o) <= 1e-6, (b, np.linalg.norm(ray_g - ray_o))
    assert same >= min_same * len(res_o), same


def sparse_cases(kind, count=6):
    """Planted infeasible LPs whose K fits the register kernel (m <= 32, n <= 64, rows/cols <= 8)."""
    out = []
    for s in range(200):
        lp = lpgen.g_infeasible(kind, s, m1=10, m2=3, n=20, density=0.15)
        if np.diff(lp.row_ptr).max() <= 8 and np.bincount(lp.col_idx, minlength=lp.n).max() <= 8:
            out.append(lp)
        if len(out) == count:
            return out
    raise AssertionError("not enough register-kernel cases")


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("kind", ["primal", "dual"])
@pytest.mark.parametrize("path", [mp.PATH_AUTO, mp.PATH_INSTANCE])
def test_single_instances(path, kind, alg, rule):
    """One LP per handle; AUTO picks the register kernel for these shapes."""
    for lp in sparse_cases(kind):
        ro = oracle.solve(lp, alg, iteration_limit=LIMIT, step_rule=rule)
        with mp.Solver(mp.Problem.from_lp(lp)) as s:
            rg = s.solve(algorithm=alg, iteration_limit=LIMIT, step_rule=rule, path=path)
            x, y, lam = s.solution()
        compare(lp, [rg], [x], [y], [ro], [ro["x"]], [ro["y"]], min_same=same_frac(rule))
        if rg["status"] == PI:  # reduced costs of the ray: -K'd_y
            assert np.allclose(lam, -(lp.dense_K().T @ y), atol=1e-9)


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("alg", ALGS)
def test_batch_with_mixed_statuses(alg, rule):
    """A batch sharing K where half the cost vectors make the LP unbounded."""
    lp = sparse_cases("dual", 1)[0]
    j = int(np.nonzero(~np.isfinite(lp.u))[0][0])
    rng = np.random.default_rng(5)
    C = lp.c + 0.1 * rng.normal(size=(64, lp.n))
    C[::2, j] = np.abs(C[::2, j]) + 1.0       # even: bounded -> OPTIMAL
    C[1::2, j] = -np.abs(C[1::2, j]) - 0.5    # odd: unbounded -> DUAL_INFEASIBLE
    for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
        res = bs.solve(algorithm=alg, iteration_limit=LIMIT, step_rule=rule, path=path)
        X, Y = bs.solutions()
        bs.close()
        Xo, Yo, ro = oracle.solve_batch(lp, C, None, alg, iteration_limit=LIMIT, step_rule=rule)
        for b in range(64):
            assert ro[b]["status"] == (oracle.OPTIMAL if b % 2 == 0 else DI), (b, ro[b]["status"])
        compare(lp, res, X, Y, ro, Xo, Yo, min_same=0.9 * same_frac(rule))


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("kind", ["primal", "dual"])
def test_dmma_dense_batch(kind, alg, rule):
    lp = lpgen.g_infeasible(kind, 1, m1=20, m2=6, n=40, dense=True)
    rng = np.random.default_rng(7)
    C = lp.c + 0.05 * rng.normal(size=(16, lp.n))
    if kind == "dual":
        j = int(np.nonzero(~np.isfinite(lp.u))[0][0])
        C[:, j] = -np.abs(C[:, j]) - 0.5
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    res = bs.solve(algorithm=alg, iteration_limit=LIMIT, step_rule=rule, path=mp.PATH_DMMA)
    X, Y = bs.solutions()
    bs.close()
    Xo, Yo, ro = oracle.solve_batch(lp, C, None, alg, iteration_limit=LIMIT, step_rule=rule)
    compare(lp, res, X, Y, ro, Xo, Yo, min_same=0.9 * same_frac(rule))
    if not (kind == "primal" and alg == "r2" and rule == "adaptive"):
        assert all(r["status"] == want_status(kind) for r in res)


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("kind", ["primal", "dual"])
def test_grid_and_sharded_paths(kind, alg, rule):
    """The persistent grid kernel and the row-sharded engine (1 and 3 virtual shards)."""
    lps = [lpgen.g_infeasible(kind, s) for s in range(4)]
    for lp in lps:
        ro = oracle.solve(lp, alg, iteration_limit=LIMIT, step_rule=rule)
        with mp.Solver(mp.Problem.from_lp(lp)) as s:
            rg = s.solve(algorithm=alg, iteration_limit=LIMIT, step_rule=rule, path=mp.PATH_GRID)
            x, y, _ = s.solution()
        compare(lp, [rg], [x], [y], [ro], [ro["x"]], [ro["y"]], min_same=same_frac(rule))
        for shards in (1, 3):
            with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards) as s:
                rs = s.solve(algorithm=alg, iteration_limit=LIMIT, step_rule=rule)
                xs, ys, _ = s.solution()
            compare(lp, [rs], [xs], [ys], [ro], [ro["x"]], [ro["y"]], min_same=same_frac(rule))


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("alg", ALGS)
def test_spec_examples(alg, rule):
    """S:630 acceptance #7 examples on the GPU, same verdicts as the oracle."""
    for lp in (spec_primal_infeasible(), spec_dual_infeasible()):
        ro = oracle.solve(lp, alg, iteration_limit=LIMIT, step_rule=rule)
        with mp.Solver(mp.Problem.from_lp(lp)) as s:
            rg = s.solve(algorithm=alg, iteration_limit=LIMIT, step_rule=rule)
            x, y, _ = s.solution()
        assert rg["status"] == ro["status"] or (ro["status"] == oracle.ITERATION_LIMIT
                                                and rg["status"] == oracle.NUMERICAL_ERROR)
        check_rays(lp, rg["status"], x, y)


def test_tolerance_off_disables_detection():
    lp = spec_dual_infeasible()
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        r = s.solve(algorithm="ra", iteration_limit=640, eps_dual_infeasible=-1.0)
    assert r["status"] == mp.LP_ITERATION_LIMIT
