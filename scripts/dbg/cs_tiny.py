import sys; sys.path.insert(0, '.')
import numpy as np, lpgen
import paper_2412_09734_b200 as mp
lp, C = lpgen.g_grid(batch=256, seed=11)
for alg in ("ra", "r2"):
    for K in (1, 2, 3, 8, 64, 65, 200):
        out = {}
        for path in (mp.PATH_AUTO, mp.PATH_INSTANCE):
            bs = mp.BatchSolver(mp.Problem.from_lp(lp), C)
            res = bs.solve(algorithm=alg, path=path, step_rule="constant", eps_abs=0.0, eps_rel=0.0, iteration_limit=K)
            X, Y = bs.solutions()
            bs.close()
            out[path] = (res, X, Y)
        a, b = out[mp.PATH_AUTO], out[mp.PATH_INSTANCE]
        print(alg, K, "eta", a[0][0]["eta"], b[0][0]["eta"], "dX", np.abs(a[1]-b[1]).max(), "dY", np.abs(a[2]-b[2]).max(),
              "restarts eq", np.array_equal(a[0]["restarts"], b[0]["restarts"]), "omega eq", np.array_equal(a[0]["omega"], b[0]["omega"]))
