import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, torch
import paper_2412_09734_b200 as mp
lp, C, Q, obj = lpgen.g_dense(200, 400, batch=256, seed=3)
dev = torch.device("cuda", 0)
bs = mp.BatchSolver(mp.Problem.from_lp(lp).to(dev), torch.as_tensor(C, device=dev), torch.as_tensor(Q, device=dev))
for alg in ("ra", "r2"):
    for cf in (64, 1024):
        bs.solve(algorithm=alg, path=mp.PATH_DMMA, iteration_limit=1024, eps_abs=0.0, eps_rel=0.0, check_frequency=cf)
        r = bs.solve(algorithm=alg, path=mp.PATH_DMMA, iteration_limit=1024, eps_abs=0.0, eps_rel=0.0, check_frequency=cf)
        print(alg, "check_freq", cf, "ms", round(r[0]["solve_seconds"] * 1e3, 3), "attempts max", r["attempts"].max())
