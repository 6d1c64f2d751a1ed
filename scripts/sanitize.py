"""Small solves on every kernel path, for compute-sanitizer (racecheck / synccheck / memcheck):
the register batch kernel, the CTA-per-instance kernel, the grid (cooperative) kernel with the
two-pass split and the lean sweeps, the DMMA cluster kernel, the row-sharded engine (2 virtual
shards) and the setup kernels.  Exits non-zero if a solve is not OPTIMAL."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

os.environ["MPAX_GRID_SPLIT"] = "1"     # exercise the two-pass phase B on a small LP
ok = True
lp, C = lpgen.g_grid(batch=64)
for alg in ("ra", "r2"):
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
    r = bs.solve(algorithm=alg)
    bs.solutions()
    bs.close()
    ok &= bool((r["status"] == mp.LP_OPTIMAL).all())
    print("tiny", alg, int(r["iterations"].max()), flush=True)
small = lpgen.g_rand(300, 600, 8, seed=3)
for path, name in ((mp.PATH_INSTANCE, "instance"), (mp.PATH_GRID, "grid")):
    for alg in ("ra", "r2"):
        with mp.Solver(mp.Problem.from_lp(small)) as s:
            r = s.solve(algorithm=alg, path=path, iteration_limit=256, eps_abs=1e-3, eps_rel=1e-3)
            s.solution()
        print(name, alg, r["status"], r["iterations"], flush=True)
dlp, DC, DQ, _ = lpgen.g_dense(24, 40, batch=16, seed=5)
for alg in ("ra", "r2"):
    bs = mp.BatchSolver(mp.Problem.from_lp(dlp), DC, DQ)
    r = bs.solve(algorithm=alg, path=mp.PATH_DMMA, iteration_limit=256, eps_abs=1e-3, eps_rel=1e-3)
    bs.close()
    print("dmma", alg, int(r["iterations"].max()), flush=True)
with mp.ShardedSolver(mp.Problem.from_lp(small), virtual_shards=2) as s:
    r = s.solve(algorithm="ra", iteration_limit=128, eps_abs=1e-3, eps_rel=1e-3)
    print("sharded", r["status"], r["iterations"], flush=True)
sys.exit(0 if ok else 1)
