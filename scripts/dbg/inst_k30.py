import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, torch
import paper_2412_09734_b200 as mp
lp = lpgen.warcraft_lp(30); C = lpgen.warcraft_costs(30, 70, seed=30)
dev = torch.device("cuda", 0)
bs = mp.BatchSolver(mp.Problem.from_lp(lp).to(dev), torch.as_tensor(C, device=dev))
for i in range(2):
    r = bs.solve(algorithm="ra", iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
print(1e6 * r[0]["solve_seconds"] / r["attempts"].max())
