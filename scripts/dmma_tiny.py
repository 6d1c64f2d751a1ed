"""Smallest DMMA-path run (for compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m, n, B = int(os.environ.get("DM", 12)), int(os.environ.get("DN", 20)), int(os.environ.get("DB", 8))
lp, C, Q, obj = lpgen.g_dense(m, n, batch=B, seed=5)
bs = mp.BatchSolver(mp.Problem.from_lp(lp), C, Q)
res = bs.solve(algorithm=os.environ.get("DALG", "ra"), path=mp.PATH_DMMA, iteration_limit=int(os.environ.get("DK", 1)),
               eps_abs=1e-13, eps_rel=1e-13)
print(res["status"], res["attempts"], res["primal_objective"][:3])
