import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, oracle
import paper_2412_09734_b200 as mp
lp, C = lpgen.g_grid(batch=256, seed=11)
om = {}
for rule in ("adaptive", "constant"):
    for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
        bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
        res = bs.solve(algorithm="ra", path=path, step_rule=rule, eps_abs=0.0, eps_rel=0.0, iteration_limit=1)
        bs.close()
        om[(rule, path)] = res["omega"].copy()
        print(rule, path, res["status"][:10], res["iterations"][:10])
ref = om[("adaptive", 0)]
for k, v in om.items():
    d = np.nonzero(v != ref)[0]
    print(k, len(d), d[:10], v[d[:3]], ref[d[:3]])
