"""Drive the grid path twice on C4 (G-RAND(1e5, 2e5, 20, seed 4)) or, PROF_M=5000000, C5 (seed 5)
for profiling; PROF_PREC=fp32 for fp32 storage."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("PROF_M", "100000"))
alg = os.environ.get("PROF_ALG", "ra")
K = int(os.environ.get("PROF_K", "64"))
t0 = time.time()
lp = lpgen.g_rand(m, 2 * m, 20, seed=int(os.environ.get("PROF_SEED", "4" if m < 1_000_000 else "5")))
prec = os.environ.get("PROF_PREC", "fp64")
print("gen", time.time() - t0, flush=True)
with mp.Solver(mp.Problem.from_lp(lp)) as s:
    for rep in range(2):
        r = s.solve(algorithm=alg, path=mp.PATH_GRID, iteration_limit=K, eps_abs=0.0, eps_rel=0.0, precision=prec)
        print(rep, r["status"], r["iterations"], r["attempts"], r["solve_seconds"] * 1e3, "ms",
              r["solve_seconds"] * 1e6 / r["attempts"], "us/attempt", flush=True)
if os.environ.get("PROF_SHARDED"):
    with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=1) as s:
        for rep in range(2):
            r = s.solve(algorithm=alg, iteration_limit=K, eps_abs=0.0, eps_rel=0.0)
            print("sharded-1", rep, r["status"], r["iterations"], r["attempts"], r["solve_seconds"] * 1e3, "ms",
                  r["solve_seconds"] * 1e6 / r["attempts"], "us/attempt", flush=True)
