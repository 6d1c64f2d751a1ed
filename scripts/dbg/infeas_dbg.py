import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, oracle
import paper_2412_09734_b200 as mp
from tests.test_gpu_infeasibility import sparse_cases
for kind in ("primal", "dual"):
    for alg in ("ra", "r2"):
        for rule in ("adaptive", "constant"):
            row = []
            for lp in sparse_cases(kind):
                ro = oracle.solve(lp, alg, iteration_limit=10000, step_rule=rule)
                with mp.Solver(mp.Problem.from_lp(lp)) as s:
                    rg = s.solve(algorithm=alg, iteration_limit=10000, step_rule=rule)
                    # trajectory with detection off at K = 256
                    r1 = s.solve(algorithm=alg, iteration_limit=256, step_rule=rule, eps_primal_infeasible=-1.0, eps_dual_infeasible=-1.0, eps_abs=0.0, eps_rel=0.0)
                    x1, y1, _ = s.solution()
                o1 = oracle.solve(lp, alg, iteration_limit=256, step_rule=rule, eps_primal_infeasible=-1.0, eps_dual_infeasible=-1.0, eps_abs=0.0, eps_rel=0.0)
                dx = np.linalg.norm(x1 - o1["x"]) / max(np.linalg.norm(o1["x"]), 1e-300)
                row.append((int(ro["status"]), int(ro["iterations"]), int(rg["status"]), int(rg["iterations"]), r1["attempts"] == o1["attempts"], f"{dx:.1e}"))
            print(kind, alg, rule, row)
