"""Host wall-clock breakdown of one C2 bench step (create / solve / get / destroy)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

lp, C = lpgen.g_grid(batch=1024, seed=2)
dev = torch.device("cuda", 0)
for mem in ("device", "host"):
    prob = mp.Problem.from_lp(lp)
    Cx = C
    if mem == "device":
        prob = prob.to(dev)
        Cx = torch.as_tensor(C, device=dev)
    X = torch.empty((1024, lp.n), dtype=torch.float64, device=dev) if mem == "device" else np.zeros((1024, lp.n))
    Y = torch.empty((1024, lp.m), dtype=torch.float64, device=dev) if mem == "device" else np.zeros((1024, lp.m))
    kind = mp.LP_DEVICE if mem == "device" else mp.LP_HOST
    acc = np.zeros(4)
    for it in range(60):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bs = mp.BatchSolver(prob, Cx)
        t1 = time.perf_counter()
        res = bs.solve(algorithm="ra")
        t2 = time.perf_counter()
        bs.solutions(memory=kind, X=X, Y=Y)
        t3 = time.perf_counter()
        bs.close()
        t4 = time.perf_counter()
        if it >= 10:
            acc += [t1 - t0, t2 - t1, t3 - t2, t4 - t3]
    acc /= 50
    print(mem, "create %.3f ms  solve %.3f ms (kernel %.3f)  get %.3f ms  destroy %.3f ms" % (
        acc[0] * 1e3, acc[1] * 1e3, res[0]["solve_seconds"] * 1e3, acc[2] * 1e3, acc[3] * 1e3), flush=True)
