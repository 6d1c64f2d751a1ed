"""GPU parity of the row-sharded engine against the CPU oracle.
One GPU: `virtual` shards (p row blocks on one device, fixed-order device sum in
place of NCCL) exercise the partitioned arithmetic; a real 1-rank NCCL
communicator exercises the NCCL plumbing."""
import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2412_09734_b200 as mp  # noqa: E402
from tests.test_gpu_parity import obj_tol, oracle_stability, rel  # noqa: E402

ALGS = ["ra", "r2"]


def _long_cols(seed=9):
    """K' of a G-POWERLAW pattern: columns of up to ~400 entries (the long-row path of the K~'y
    SpMV), rows short; a box keeps every fixed-K trajectory bounded."""
    p = lpgen.g_powerlaw(400, 800, 12, seed=seed)
    K = np.zeros((p.m, p.n))
    rows = np.repeat(np.arange(p.m), np.diff(p.row_ptr))
    K[rows, p.col_idx] = p.val
    KT = K.T                                                   # 800 x 400
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1, 1, KT.shape[1])
    q = KT @ x0
    return lpgen.stack(rng.normal(size=KT.shape[1]), G=KT[:400], h=q[:400] - 1.0, A=KT[400:], b=q[400:],
                       l=np.full(KT.shape[1], -5.0), u=np.full(KT.shape[1], 5.0))


# "powerlaw": rows of up to 421 entries, "longcols": columns of up to ~400 -- the full-chunk
# (long-row) path of the warp-tile SpMV on each side (the kernels' LR instantiations)
LONG = [("powerlaw", lpgen.g_powerlaw(2000, 4000, 12, seed=9)), ("longcols", _long_cols())]
CASES = [("C1", lpgen.g_rand(50, 100, 10, seed=1)), ("mid", lpgen.g_rand(3000, 5000, 12, seed=3)),
         ("tiny", lpgen.tiny_spec())] + LONG


def sharded(lp, alg, shards, **kw):
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards) as s:
        r = s.solve(algorithm=alg, **kw)
        x, y, lam = s.solution()
    r.update(x=x, y=y, lam=lam)
    return r


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 2, 64])
@pytest.mark.parametrize("shards", [1, 2, 3])
@pytest.mark.parametrize("name,lp", CASES)
def test_sharded_fixed_K(alg, K, shards, name, lp):
    if shards > lp.m:
        pytest.skip("more shards than rows")
    ro, stable, drift = oracle_stability(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    rg = sharded(lp, alg, shards, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    if not stable:
        pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rel(rg["x"], ro["x"]) <= tol
    if lp.m:
        assert rel(rg["y"], ro["y"]) <= tol


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 4])
@pytest.mark.parametrize("name,lp", CASES[:2])
def test_sharded_full_solve(alg, shards, name, lp):
    ro, stable, drift = oracle_stability(lp, alg)
    rg = sharded(lp, alg, shards)
    assert rg["status"] == mp.LP_OPTIMAL and rg["rel_kkt"] <= 1e-4
    if stable:
        assert rg["iterations"] == ro["iterations"] and rg["restarts"] == ro["restarts"]
        assert abs(rg["primal_objective"] - ro["primal_objective"]) <= obj_tol(ro) * (1 + abs(ro["primal_objective"]))
    k = oracle.kkt_original(lp, rg["x"], rg["y"])
    assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.q))
    assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.c))
    assert abs(rg["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))


def test_nccl_one_rank_equals_virtual_one_shard():
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    uid = mp.nccl_unique_id()
    comm = mp.nccl_comm_init(1, uid, 0)
    try:
        with mp.ShardedSolver(mp.Problem.from_lp(lp), 0, lp.m1, lp.m2, comm=comm, rank=0, nranks=1) as s:
            a = s.solve(algorithm="r2", iteration_limit=200, eps_abs=0.0, eps_rel=0.0)
            xa, ya, _ = s.solution()
    finally:
        mp.nccl_comm_destroy(comm)
    b = sharded(lp, "r2", 1, iteration_limit=200, eps_abs=0.0, eps_rel=0.0)
    assert a["attempts"] == b["attempts"] and np.array_equal(xa, b["x"]) and np.array_equal(ya, b["y"])


def test_sharded_local_rows_api_matches_virtual():
    """A 'rank' built from python-side local_rows(row_partition(...)) solves its
    block exactly like the library's own virtual split (same cut rule)."""
    lp = lpgen.g_rand(400, 700, 8, seed=6)
    prob = mp.Problem.from_lp(lp)
    cuts = mp.row_partition(lp.row_ptr, 3)
    assert cuts[0] == 0 and cuts[-1] == lp.m and all(a <= b for a, b in zip(cuts, cuts[1:]))
    loc = mp.local_rows(prob, cuts[1], cuts[2])
    assert loc.m1 == max(0, min(lp.m1 - cuts[1], cuts[2] - cuts[1]))
    K = lp.dense_K()
    Kl = lpgen.LP(loc.n, loc.m1, loc.m2, np.asarray(loc.row_ptr), np.asarray(loc.col_idx),
                  np.asarray(loc.values), lp.c, np.asarray(loc.q), lp.l, lp.u).dense_K()
    assert np.array_equal(Kl, K[cuts[1]:cuts[2]])


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 3])
@pytest.mark.parametrize("name,lp", CASES[:2])
def test_sharded_two_pass_rows(alg, shards, name, lp, monkeypatch):
    """The rows step over the column halves of each K~_g (forced on; by default only past the
    L2 gather knee) against the oracle at fixed K."""
    monkeypatch.setenv("MPAX_GRID_SPLIT", "1")
    ro, stable, drift = oracle_stability(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=64)
    rg = sharded(lp, alg, shards, eps_abs=0.0, eps_rel=0.0, iteration_limit=64)
    if not stable:
        pytest.skip("ill-conditioned at this K")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rel(rg["x"], ro["x"]) <= tol and rel(rg["y"], ro["y"]) <= tol


# ---- column sharding (the axis chosen by min(m, n); reading 33) ----
COL_CASES = [("C1", lpgen.g_rand(50, 100, 10, seed=1)), ("wide", lpgen.g_rand(700, 9000, 30, seed=8)),
             ("tiny", lpgen.tiny_spec())] + LONG


def sharded_cols(lp, alg, shards, axis="cols", **kw):
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards, axis=axis) as s:
        r = s.solve(algorithm=alg, **kw)
        x, y, lam = s.solution()
    r.update(x=x, y=y, lam=lam)
    return r


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 2])
@pytest.mark.parametrize("name,lp", COL_CASES[:2] + LONG)
def test_sharded_two_pass_cols(alg, shards, name, lp, monkeypatch):
    """Column mode's K~_g x'_g over the column halves of each shard (forced on; by default only
    past the L2 gather knee) against the oracle at fixed K."""
    monkeypatch.setenv("MPAX_GRID_SPLIT", "1")
    ro, stable, drift = oracle_stability(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=64)
    rg = sharded_cols(lp, alg, shards, eps_abs=0.0, eps_rel=0.0, iteration_limit=64)
    if not stable:
        pytest.skip("ill-conditioned at this K")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rel(rg["x"], ro["x"]) <= tol and rel(rg["y"], ro["y"]) <= tol


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 2, 64])
@pytest.mark.parametrize("shards", [1, 2, 3])
@pytest.mark.parametrize("name,lp", COL_CASES)
def test_cols_fixed_K(alg, K, shards, name, lp):
    if shards > lp.n:
        pytest.skip("more shards than columns")
    ro, stable, drift = oracle_stability(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    rg = sharded_cols(lp, alg, shards, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    if not stable:
        pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rg[key] == ro[key], (key, rg[key], ro[key])
    assert rel(rg["x"], ro["x"]) <= tol
    assert rel(rg["lam"], ro["lam"]) <= max(1e-8, 1e3 * drift)
    if lp.m:
        assert rel(rg["y"], ro["y"]) <= tol


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("shards", [1, 4])
@pytest.mark.parametrize("name,lp", COL_CASES[:2])
def test_cols_full_solve(alg, shards, name, lp):
    ro, stable, drift = oracle_stability(lp, alg)
    rg = sharded_cols(lp, alg, shards)
    assert rg["status"] == mp.LP_OPTIMAL and rg["rel_kkt"] <= 1e-4
    if stable:
        assert rg["iterations"] == ro["iterations"] and rg["restarts"] == ro["restarts"]
        assert abs(rg["primal_objective"] - ro["primal_objective"]) <= obj_tol(ro) * (1 + abs(ro["primal_objective"]))
    k = oracle.kkt_original(lp, rg["x"], rg["y"])
    assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.q))
    assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.c))
    assert abs(rg["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))


def test_axis_auto_and_refusals():
    wide = lpgen.g_rand(50, 100, 10, seed=1)          # m < n: columns
    a = sharded_cols(wide, "r2", 2, axis="auto", iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
    b = sharded_cols(wide, "r2", 2, axis="cols", iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
    assert a["attempts"] == b["attempts"] and np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
    tall = lpgen.g_rand(100, 60, 8, seed=2)           # m >= n: rows
    a = sharded_cols(tall, "r2", 2, axis="auto", iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
    b = sharded(tall, "r2", 2, iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
    assert a["attempts"] == b["attempts"] and np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])


@pytest.mark.parametrize("alg", ALGS)
def test_cols_polish_and_warm_start(alg):
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    ro = oracle.solve(lp, alg, eps_abs=1e-2, eps_rel=1e-2, feasibility_polishing=True)
    rg = sharded_cols(lp, alg, 3, eps_abs=1e-2, eps_rel=1e-2, feasibility_polishing=1)
    assert rg["status"] == ro["status"] == mp.LP_OPTIMAL and rg["polish"] == ro["polish"] == 1
    k = oracle.kkt_original(lp, rg["x"], rg["y"])
    assert k["pres"] <= (1 + 1e-9) * 1e-6 * (1 + np.linalg.norm(lp.q))
    assert k["dres"] <= (1 + 1e-9) * 1e-6 * (1 + np.linalg.norm(lp.c))
    assert rg["primal_objective"] == pytest.approx(float(lp.c @ rg["x"]), rel=1e-12)
    rng = np.random.default_rng(2)
    x0, y0 = rng.normal(size=lp.n), rng.normal(size=lp.m)
    ro = oracle.solve(lp, alg, x0=x0, y0=y0, iteration_limit=64, eps_abs=0, eps_rel=0)
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=2, axis="cols") as s:
        rg = s.solve(x0, y0, algorithm=alg, iteration_limit=64, eps_abs=0.0, eps_rel=0.0)
        x, y, _ = s.solution()
    assert rg["attempts"] == ro["attempts"] and rel(x, ro["x"]) <= 1e-9 and rel(y, ro["y"]) <= 1e-9


@pytest.mark.parametrize("axis", ["rows", "cols"])
def test_graph_replay_matches_direct(axis, monkeypatch):
    """The attempt chunks replayed from the CUDA graph (default) and enqueued kernel by kernel
    (MPAX_SHARDED_GRAPH=0) are the same computation: identical results and kernel counts."""
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)

    def run():
        before = mp.launch_count()
        with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=2, axis=axis) as s:
            r = s.solve(algorithm="r2", iteration_limit=300, eps_abs=0.0, eps_rel=0.0)
            x, y, _ = s.solution()
        return r, x, y, mp.launch_count() - before

    a = run()
    monkeypatch.setenv("MPAX_SHARDED_GRAPH", "0")
    b = run()
    assert a[0]["attempts"] == b[0]["attempts"] and a[0]["restarts"] == b[0]["restarts"]
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert a[3] == b[3]


# ---- exchange variant B of the row engine (reduce-scatter + all-gather) ----
@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("K", [1, 64])
@pytest.mark.parametrize("shards", [1, 2, 3])
@pytest.mark.parametrize("name,lp", CASES)
def test_variant_b_fixed_K(alg, K, shards, name, lp):
    if shards > lp.m:
        pytest.skip("more shards than rows")
    ro, stable, drift = oracle_stability(lp, alg, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    rb = sharded(lp, alg, shards, eps_abs=0.0, eps_rel=0.0, iteration_limit=K, sharded_exchange=1)
    ra = sharded(lp, alg, shards, eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
    if not stable:
        pytest.skip("ill-conditioned at this K: the oracle's own counts move under a 1-ulp perturbation")
    tol = max(1e-9, 100 * drift)
    for key in ("status", "iterations", "attempts", "restarts"):
        assert rb[key] == ro[key] == ra[key], (key, rb[key], ro[key], ra[key])
    for v in ("x", "y", "lam"):
        if v == "y" and not lp.m:
            continue
        assert rel(rb[v], ro[v]) <= (tol if v != "lam" else max(1e-8, 1e3 * drift))
        assert rel(rb[v], ra[v]) <= max(1e-10, 100 * drift)   # A, B differ in the order of the column sums


@pytest.mark.parametrize("alg", ALGS)
def test_variant_b_full_solve_and_polish(alg):
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    rb = sharded(lp, alg, 3, sharded_exchange=1)
    assert rb["status"] == mp.LP_OPTIMAL and rb["rel_kkt"] <= 1e-4
    k = oracle.kkt_original(lp, rb["x"], rb["y"])
    assert k["pres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.q))
    assert k["dres"] <= (1 + 1e-6) * (1e-4 + 1e-4 * np.linalg.norm(lp.c))
    assert abs(rb["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star))
    small = lpgen.g_rand(50, 100, 10, seed=1)
    rp = sharded(small, alg, 2, eps_abs=1e-2, eps_rel=1e-2, feasibility_polishing=1, sharded_exchange=1)
    assert rp["status"] == mp.LP_OPTIMAL and rp["polish"] == 1
    k = oracle.kkt_original(small, rp["x"], rp["y"])
    assert k["pres"] <= (1 + 1e-9) * 1e-6 * (1 + np.linalg.norm(small.q))
    assert k["dres"] <= (1 + 1e-9) * 1e-6 * (1 + np.linalg.norm(small.c))
    assert rp["primal_objective"] == pytest.approx(float(small.c @ rp["x"]), rel=1e-12)


@pytest.mark.parametrize("shards", [2, 3])
def test_chunked_exchange_matches_unchunked(shards, monkeypatch):
    """Variant A with the K~_g'y partials summed and all-reduced chunk by chunk on a second stream
    (MPAX_SHARDED_CHUNKS): every element is the same sum in the same shard order, so the solve is
    bitwise the unchunked one (graph replay included)."""
    lp = lpgen.g_rand(3000, 5000, 12, seed=3)
    monkeypatch.setenv("MPAX_SHARDED_CHUNKS", "1")
    a = sharded(lp, "r2", shards, iteration_limit=300, eps_abs=0.0, eps_rel=0.0)
    monkeypatch.setenv("MPAX_SHARDED_CHUNKS", "4")
    b = sharded(lp, "r2", shards, iteration_limit=300, eps_abs=0.0, eps_rel=0.0)
    assert a["attempts"] == b["attempts"] and a["restarts"] == b["restarts"]
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])


def test_nccl_one_rank_columns_equals_virtual():
    """lp_create_sharded_cols through a real 1-rank NCCL communicator (the multi-process entry
    point, its local block being the whole LP) against the virtual 1-shard column engine."""
    lp = lpgen.g_rand(700, 9000, 30, seed=8)
    prob = mp.Problem.from_lp(lp)
    loc = mp.local_cols(prob, 0, lp.n)
    uid = mp.nccl_unique_id()
    comm = mp.nccl_comm_init(1, uid, 0)
    try:
        with mp.ShardedSolver(loc, comm=comm, rank=0, nranks=1, axis="cols", global_col_offset=0,
                              n_global=lp.n) as s:
            a = s.solve(algorithm="r2", iteration_limit=200, eps_abs=0.0, eps_rel=0.0)
            xa, ya, la = s.solution()
    finally:
        mp.nccl_comm_destroy(comm)
    b = sharded_cols(lp, "r2", 1, iteration_limit=200, eps_abs=0.0, eps_rel=0.0)
    assert a["attempts"] == b["attempts"]
    assert np.array_equal(xa, b["x"]) and np.array_equal(ya, b["y"]) and np.array_equal(la, b["lam"])


@pytest.mark.slow
def test_c5_sharded_full_size_sampled():
    """C5 = G-RAND(5e6, 1e7, 20, seed 5) at its BASELINE size on the sharded engine in the launch
    configuration `bench.py --c5-sharded` (and every N > 1 run) times: a 1-rank NCCL
    communicator, by rows and by columns.  Iterates after K = 2 accepted r2HPDHG steps against the
    oracle (~30 s on the host), then a full raPDHG solve to 1e-4 checked by properties."""
    lp = lpgen.g_rand(5_000_000, 10_000_000, 20, seed=5)
    oracle.set_threads(0)
    ro = oracle.solve(lp, "r2", iteration_limit=2, eps_abs=0.0, eps_rel=0.0)
    full = mp.Problem.from_lp(lp)
    for axis in ("rows", "cols"):
        if axis == "cols":
            loc, kw = mp.local_cols(full, 0, lp.n).to("cuda:0"), dict(axis="cols", n_global=lp.n)
        else:
            loc, kw = full.to("cuda:0"), dict(m1_global=lp.m1, m2_global=lp.m2)
        comm = mp.nccl_comm_init(1, mp.nccl_unique_id(), 0)
        try:
            with mp.ShardedSolver(loc, comm=comm, rank=0, nranks=1, **kw) as s:
                rg = s.solve(algorithm="r2", iteration_limit=2, eps_abs=0.0, eps_rel=0.0)
                x, y, _ = s.solution()
                assert rg["attempts"] == ro["attempts"], axis
                assert rel(x, ro["x"]) <= 1e-12 and rel(y, ro["y"]) <= 1e-12, axis
                r = s.solve(algorithm="ra", iteration_limit=5000)
                x, y, _ = s.solution()
        finally:
            mp.nccl_comm_destroy(comm)
        del loc
        assert r["status"] == mp.LP_OPTIMAL and r["rel_kkt"] <= 1e-4, axis
        assert abs(r["primal_objective"] - lp.obj_star) <= 1e-3 * (1 + abs(lp.obj_star)), axis
        assert np.all(y[: lp.m1] >= 0) and np.all(x >= lp.l), axis
