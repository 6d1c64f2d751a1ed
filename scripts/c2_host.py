"""Host-side anatomy of one C2 step: wall-clock microseconds of each Python call of the step
(create, solve, solutions, close) against the step's device time, over many steps (median)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

lp, C = bench.make_workload(1024, seed=2)
dev = torch.device("cuda", 0)
prob = mp.Problem.from_lp(lp).to(dev)
Cd = torch.as_tensor(C, device=dev)
X = torch.empty((1024, lp.n), dtype=torch.float64, device=dev)
Y = torch.empty((1024, lp.m), dtype=torch.float64, device=dev)
st = torch.cuda.current_stream()
T = {k: [] for k in ("create", "solve", "solutions", "close", "step_wall", "step_dev")}
for it in range(400):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(st)
    bs = mp.BatchSolver(prob, Cd)
    t1 = time.perf_counter()
    r = bs.solve(algorithm="ra", iteration_limit=200_000)
    t2 = time.perf_counter()
    bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
    t3 = time.perf_counter()
    bs.close()
    t4 = time.perf_counter()
    b.record(st)
    torch.cuda.synchronize()
    if it >= 50:
        for k, v in zip(("create", "solve", "solutions", "close", "step_wall"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            T[k].append(v * 1e6)
        T["step_dev"].append(a.elapsed_time(b) * 1e3)
print("median us:", {k: round(float(np.median(v)), 1) for k, v in T.items()},
      "kernel us:", round(float(r["solve_seconds"][0]) * 1e6, 1))
