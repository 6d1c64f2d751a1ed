import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, torch
import paper_2412_09734_b200 as mp
lp, C = lpgen.g_grid(batch=1024, seed=2)
dev = torch.device("cuda", 0)
prob = mp.Problem.from_lp(lp).to(dev)
Cd = torch.as_tensor(C, device=dev)
for alg in ("ra", "r2"):
    for rule in ("adaptive", "constant"):
        ts = []
        t1 = []
        for rep in range(5):
            bs = mp.BatchSolver(prob, Cd)
            r1 = bs.solve(algorithm=alg, step_rule=rule, iteration_limit=1)
            r = bs.solve(algorithm=alg, step_rule=rule)
            bs.close()
            t1.append(r1[0]["solve_seconds"] * 1e3)
            ts.append(r[0]["solve_seconds"] * 1e3)
        it = r["iterations"]
        print(alg, rule, "first-solve(K=1) ms", np.round(t1, 4), "solve ms", np.round(ts, 4), "iters p50/max", np.median(it), it.max(), "att sum", r["attempts"].sum())
