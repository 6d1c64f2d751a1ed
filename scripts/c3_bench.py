"""C3 (256 dense 200x400 LPs sharing K): LPs/s of the available batch paths."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

lp, C, Q, obj = lpgen.g_dense(200, 400, batch=256, seed=3)
prob = mp.Problem.from_lp(lp).to("cuda:0")
Cd, Qd = torch.as_tensor(C, device="cuda:0"), torch.as_tensor(Q, device="cuda:0")
paths = [int(p) for p in os.environ.get("C3_PATHS", "3,1").split(",")]
for path in paths:
    for alg in ("ra", "r2"):
        bs = mp.BatchSolver(prob, Cd, Qd)
        try:
            res = bs.solve(algorithm=alg, path=path, iteration_limit=100000)
            res = bs.solve(algorithm=alg, path=path, iteration_limit=100000)
        except mp.LpError as e:
            print(path, alg, "error", e)
            continue
        t = res[0]["solve_seconds"]
        it = res["iterations"]
        ok = (res["status"] == 1).all()
        err = np.max(np.abs(res["primal_objective"] - obj) / (1 + np.abs(obj)))
        print(f"path={path} {alg}: {256 / t:9.1f} LPs/s  solve {t * 1e3:8.2f} ms  iters p50 {np.median(it):.0f} "
              f"max {it.max()}  all_optimal {ok}  max obj err {err:.2e}", flush=True)
        bs.close()
