"""Host-side cost of the C2 step's Python binding calls (per call, microseconds), with the
library's own phase marks (MPAX_HOST_TRACE=1 prints them to stderr)."""
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
T = {k: [] for k in ("stream", "opts", "create", "solve", "solutions", "close", "ctypes_noop")}
for it in range(60):
    t0 = time.perf_counter(); torch.cuda.current_stream().cuda_stream; T["stream"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); mp.default_options(algorithm="ra", iteration_limit=200000); T["opts"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); mp.lib().lp_kernel_launch_count(); T["ctypes_noop"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); bs = mp.BatchSolver(prob, Cd); T["create"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); r = bs.solve(algorithm="ra", iteration_limit=200_000); T["solve"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y); T["solutions"].append(time.perf_counter() - t0)
    t0 = time.perf_counter(); bs.close(); T["close"].append(time.perf_counter() - t0)
for k, v in T.items():
    print(f"{k:12s} median {np.median(v[10:]) * 1e6:8.1f} us")
