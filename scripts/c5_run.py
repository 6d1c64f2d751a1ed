"""C5 = G-RAND(5e6, 1e7, 20, seed 5) at full size: setup time, time to 1e-4 on the
grid path (both algorithms), achieved GB/s, and a K=2 parity sample vs the oracle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("C5_M", "5000000"))
t0 = time.time()
lp = lpgen.g_rand(m, 2 * m, 20, seed=5)
print(f"gen {time.time() - t0:.1f}s nnz {lp.nnz}", flush=True)
prob = mp.Problem.from_lp(lp).to("cuda:0")
torch.cuda.synchronize()
t0 = time.time()
s = mp.Solver(prob)
torch.cuda.synchronize()
print(f"create (validate+transpose+precondition) {time.time() - t0:.3f}s", flush=True)
res = {}
precs = os.environ.get("C5_PREC", "fp64").split(",")
for alg in os.environ.get("C5_ALGS", "ra,r2").split(","):
    for prec in precs:
        e = 8 if prec == "fp64" else 4
        for _ in range(int(os.environ.get("C5_REPS", "1"))):   # > 1: the last solve is reported (warm)
            r = s.solve(algorithm=alg, path=mp.PATH_GRID, iteration_limit=int(os.environ.get("C5_LIMIT", "4000")),
                        precision=prec)
        pair = 2 * (4 + e) * lp.nnz + 4 * (lp.m + 1) + 4 * (lp.n + 1) + e * lp.n + e * lp.m
        upd = e * (8 * lp.n + 7 * lp.m if alg == "ra" else 11 * lp.n + 11 * lp.m)
        gbs = r["iterations"] * (pair + upd) / r["solve_seconds"] / 1e9
        if prec == "fp64" or alg not in res:
            res[alg] = r
        print(f"{alg} {prec}: status {r['status']} it {r['iterations']} att {r['attempts']} restarts {r['restarts']} "
              f"time {r['solve_seconds']:.3f}s  {r['solve_seconds'] * 1e6 / r['attempts']:.0f} us/attempt  "
              f"{gbs:.0f} GB/s  rel_kkt {r['rel_kkt']:.2e}  obj err {abs(r['primal_objective'] - lp.obj_star) / (1 + abs(lp.obj_star)):.2e}",
              flush=True)
if os.environ.get("C5_ORACLE"):
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))
    for alg in os.environ.get("C5_ALGS", "ra,r2").split(","):
        t0 = time.time()
        ro = oracle.solve(lp, alg, iteration_limit=2, eps_abs=0.0, eps_rel=0.0)
        t1 = time.time()
        rg = s.solve(algorithm=alg, path=mp.PATH_GRID, iteration_limit=2, eps_abs=0.0, eps_rel=0.0)
        x, y, _ = s.solution()
        ex = np.linalg.norm(x - ro["x"]) / np.linalg.norm(ro["x"])
        ey = np.linalg.norm(y - ro["y"]) / np.linalg.norm(ro["y"])
        print(f"parity K=2 {alg}: oracle {t1 - t0:.1f}s attempts {ro['attempts']}/{rg['attempts']} "
              f"rel x {ex:.2e} rel y {ey:.2e}", flush=True)
s.close()
