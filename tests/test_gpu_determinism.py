"""Run-to-run determinism of every engine under repetition -- the race detector available on this
pool (compute-sanitizer is closed on it): a race between CTAs, warps or streams (dynamic tile
claims, per-CTA partial buffers, cluster barriers, the sharded engine's second stream and graph
replay) shows up as results that differ between identical solves.  Every engine sums in a fixed
order, so repeated solves must agree bit for bit."""
import numpy as np
import pytest

import lpgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402

REPS = 8


def _same(runs):
    r0 = runs[0]
    for r in runs[1:]:
        assert r[0] == r0[0]
        for a, b in zip(r[1:], r0[1:]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("alg", ["ra", "r2"])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_grid_repeated(alg, prec):
    lp = lpgen.g_rand(20000, 40000, 20, seed=6)
    runs = []
    with mp.Solver(mp.Problem.from_lp(lp).to("cuda")) as s:
        for _ in range(REPS):
            r = s.solve(algorithm=alg, path=mp.PATH_GRID, precision=prec, iteration_limit=400, eps_abs=0.0,
                        eps_rel=0.0)
            x, y, lam = s.solution()
            runs.append(((r["attempts"], r["restarts"]), x, y, lam))
    _same(runs)


def test_grid_long_rows_repeated():
    lp = lpgen.g_powerlaw(20000, 40000, 20, seed=9)
    runs = []
    with mp.Solver(mp.Problem.from_lp(lp).to("cuda")) as s:
        for _ in range(REPS):
            r = s.solve(algorithm="ra", path=mp.PATH_GRID, iteration_limit=300, eps_abs=0.0, eps_rel=0.0)
            x, y, lam = s.solution()
            runs.append(((r["attempts"], r["restarts"]), x, y, lam))
    _same(runs)


@pytest.mark.parametrize("alg", ["ra", "r2"])
def test_tiny_batch_repeated(alg):
    lp, C = lpgen.g_grid(batch=1024, seed=2)
    prob = mp.Problem.from_lp(lp).to("cuda")
    Cd = torch.as_tensor(C, device="cuda")
    runs = []
    for _ in range(REPS):
        bs = mp.BatchSolver(prob, Cd)
        res = bs.solve(algorithm=alg)
        X, Y = bs.solutions()
        bs.close()
        runs.append((tuple(np.asarray(res["attempts"]).tolist()), X, Y))
    _same(runs)


def test_dmma_repeated():
    lp, C, Q, _ = lpgen.g_dense(200, 400, batch=64, seed=3)
    runs = []
    for _ in range(REPS):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
        res = bs.solve(algorithm="ra", path=mp.PATH_DMMA, iteration_limit=256, eps_abs=0.0, eps_rel=0.0)
        X, Y = bs.solutions()
        bs.close()
        runs.append((tuple(np.asarray(res["attempts"]).tolist()), X, Y))
    _same(runs)


@pytest.mark.parametrize("mode", ["rows", "rows-chunked", "rows-B", "cols"])
def test_sharded_repeated(mode, monkeypatch):
    lp = lpgen.g_rand(3000, 5000, 12, seed=3) if mode != "cols" else lpgen.g_rand(700, 9000, 30, seed=8)
    if mode == "rows-chunked":
        monkeypatch.setenv("MPAX_SHARDED_CHUNKS", "4")
    kw = dict(sharded_exchange=1) if mode == "rows-B" else {}
    runs = []
    for _ in range(REPS // 2):
        with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=3,
                              axis="cols" if mode == "cols" else "rows") as s:
            r = s.solve(algorithm="r2", iteration_limit=256, eps_abs=0.0, eps_rel=0.0, **kw)
            x, y, lam = s.solution()
        runs.append(((r["attempts"], r["restarts"]), x, y, lam))
    _same(runs)
