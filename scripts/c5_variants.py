"""Per-attempt time of the grid path on a large G-RAND LP under grid-kernel knobs (environment
variables read by every grid_solve call), one LP generation for all variants.
VARIANTS="MPAX_GRID_LEAN=0;MPAX_GRID_LEAN=3" PROF_M=5000000 PROF_K=32 python scripts/c5_variants.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("PROF_M", "5000000"))
K = int(os.environ.get("PROF_K", "32"))
algs = os.environ.get("PROF_ALGS", "ra").split(",")
variants = [v for v in os.environ.get("VARIANTS", "MPAX_GRID_LEAN=3").split(";") if v]
t0 = time.time()
lp = lpgen.g_rand(m, 2 * m, 20, seed=5 if m >= 1_000_000 else 4)
print(f"gen {time.time() - t0:.1f} s nnz {lp.nnz}", flush=True)
with mp.Solver(mp.Problem.from_lp(lp)) as s:
    for rnd in range(2):
        for v in variants:
            env = dict(kv.split("=") for kv in v.split(","))
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            for alg in algs:
                r = s.solve(algorithm=alg, path=mp.PATH_GRID, iteration_limit=K, eps_abs=0.0, eps_rel=0.0)
                print(f"round {rnd} {v:28s} {alg} status {r['status']} it {r['iterations']} att {r['attempts']} "
                      f"{r['solve_seconds'] * 1e3:8.2f} ms  {r['solve_seconds'] * 1e6 / r['attempts']:8.1f} us/attempt "
                      f"obj {r['primal_objective']:.12e}", flush=True)
            for k, o in old.items():
                if o is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = o
