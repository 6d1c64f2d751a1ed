import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, torch
import paper_2412_09734_b200 as mp
lp, C = lpgen.g_grid(batch=1024, seed=2)
dev = torch.device("cuda", 0)
prob = mp.Problem.from_lp(lp).to(dev)
Cd = torch.as_tensor(C, device=dev)
for rep in range(3):
    bs = mp.BatchSolver(prob, Cd)
    r1 = bs.solve(algorithm="r2", step_rule="constant", iteration_limit=1)
    bs.close()
