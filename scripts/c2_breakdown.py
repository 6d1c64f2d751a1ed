"""Where a C2 bench step's time goes: CUDA events between the API calls of one step (create /
solve / solutions / close), host wall time of each call, and the kernel time the solve reports."""
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
gpu = np.zeros(4)
host = np.zeros(4)
kern = 0.0
N = 200
for it in range(N + 10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    h = [time.perf_counter()]
    ev[0].record(st)
    bs = mp.BatchSolver(prob, Cd)
    ev[1].record(st); h.append(time.perf_counter())
    r = bs.solve(algorithm="ra", iteration_limit=200_000)
    ev[2].record(st); h.append(time.perf_counter())
    bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
    ev[3].record(st); h.append(time.perf_counter())
    bs.close()
    ev[4].record(st); h.append(time.perf_counter())
    torch.cuda.synchronize()
    if it >= 10:
        gpu += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        host += np.diff(h) * 1e3
        kern += r[0]["solve_seconds"] * 1e3
gpu /= N; host /= N; kern /= N
names = ["create", "solve", "solutions", "close"]
print("event ms :", "  ".join(f"{n} {v:.4f}" for n, v in zip(names, gpu)), f" total {gpu.sum():.4f}")
print("host  ms :", "  ".join(f"{n} {v:.4f}" for n, v in zip(names, host)), f" total {host.sum():.4f}")
print(f"solve_seconds (kernel events inside lp_solve_batch) {kern:.4f} ms")
