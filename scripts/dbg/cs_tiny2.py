import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, oracle
import paper_2412_09734_b200 as mp
lp, C = lpgen.g_grid(batch=8, seed=11)
for rule in ("adaptive", "constant"):
    for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
        res = bs.solve(algorithm="ra", path=path, step_rule=rule, eps_abs=0.0, eps_rel=0.0, iteration_limit=1)
        bs.close()
        print(rule, path, [float(r["omega"]).hex() for r in res[:3]], [float(r["eta"]).hex() for r in res[:2]])
Xo, Yo, ro = oracle.solve_batch(lp, C[:3], None, "ra", eps_abs=0.0, eps_rel=0.0, iteration_limit=1, step_rule=1)
print("oracle", [float(r["omega"]).hex() for r in ro])
