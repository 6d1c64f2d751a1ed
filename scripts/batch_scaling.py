"""C2-shaped throughput vs batch size (context for serving; the bench headline stays at
BASELINE's 1024): create + solve + get + destroy per step, device-resident inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

dev = torch.device("cuda", 0)
for B in (1024, 4096, 16384, 65536):
    lp, C = lpgen.g_grid(batch=B, seed=2)
    prob = mp.Problem.from_lp(lp).to(dev)
    Cd = torch.as_tensor(C, device=dev)
    X = torch.empty((B, lp.n), dtype=torch.float64, device=dev)
    Y = torch.empty((B, lp.m), dtype=torch.float64, device=dev)
    for alg, rule in (("ra", "adaptive"), ("r2", "constant")):
        times = []
        for rep in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bs = mp.BatchSolver(prob, Cd)
            res = bs.solve(algorithm=alg, step_rule=rule)
            bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
            bs.close()
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
        ms = min(times)
        it = res["iterations"]
        print(f"B={B:6d} {alg}/{rule:8s} step {ms:8.3f} ms  {B / ms * 1e3 / 1e6:6.3f} M LPs/s  "
              f"max it {it.max()}  all optimal {(res['status'] == mp.LP_OPTIMAL).all()}", flush=True)
