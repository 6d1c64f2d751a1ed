"""Where does a GPU trajectory leave the oracle's?  Solves one LP of the C2 batch to fixed K
(K = 64, 128, ...) on the GPU (the batch's register kernel) and with the oracle (plain and FMA
builds) and prints the relative distance of the iterates at each K.  A smooth, geometric growth
from ~1e-16 is rounding amplified by the dynamics (reading 30); a jump is a discrepancy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import lpgen  # noqa: E402
import oracle  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

b = int(os.environ.get("INST", 986))
alg = os.environ.get("ALG", "r2")
lp, C = lpgen.g_grid(batch=1024, seed=2)
lpb = lp.with_costs(c=C[b])


def rel(a, c):
    return float(np.linalg.norm(a - c) / max(np.linalg.norm(c), 1e-300))


full = oracle.solve(lpb, alg)
print(f"instance {b} {alg}: oracle full solve {full['iterations']} it, obj {full['primal_objective']:.12f}")
for K in list(range(64, full["iterations"] + 1, 64)):
    kw = dict(eps_abs=1e-13, eps_rel=1e-13, iteration_limit=K)
    ro = oracle.solve(lpb, alg, **kw)
    rf = oracle.solve(lpb, alg, fma=True, **kw)
    bs = mp.BatchSolver(mp.Problem.from_lp(lp), C[b:b + 1].copy())
    rg = bs.solve(algorithm=alg, **kw)
    X, Y = bs.solutions()
    bs.close()
    print(f"K {K:5d}  gpu-oracle x {rel(X[0], ro['x']):.2e} y {rel(Y[0], ro['y']):.2e}  att {rg[0]['attempts']}/{ro['attempts']}"
          f" rs {rg[0]['restarts']}/{ro['restarts']}  | fma-oracle x {rel(rf['x'], ro['x']):.2e} y {rel(rf['y'], ro['y']):.2e}"
          f" att {rf['attempts']}", flush=True)
