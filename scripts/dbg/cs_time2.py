import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, torch
import paper_2412_09734_b200 as mp
lp, C = lpgen.g_grid(batch=1024, seed=2)
dev = torch.device("cuda", 0)
prob = mp.Problem.from_lp(lp).to(dev)
Cd = torch.as_tensor(C, device=dev)
for alg in ("ra", "r2"):
    for rule in ("adaptive", "constant"):
        bs = mp.BatchSolver(prob, Cd)
        bs.solve(algorithm=alg, step_rule=rule, iteration_limit=1)
        ts = []
        for rep in range(3):
            r = bs.solve(algorithm=alg, step_rule=rule, iteration_limit=1024, eps_abs=0.0, eps_rel=0.0)
            ts.append(r[0]["solve_seconds"] * 1e3)
        bs.close()
        print(alg, rule, "ms", np.round(ts, 4), "attempts max", r["attempts"].max(), "us/attempt", 1e3 * min(ts) / r["attempts"].max(), "restarts mean", r["restarts"].mean())
