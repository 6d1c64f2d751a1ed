"""C2 step timing only (bench.py's step: create + batch solve + solutions + close), for A/B runs
of the library (MPAX_LIB)."""
import os
import sys

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
alg = os.environ.get("C2_ALG", "ra")
def step():
    bs = mp.BatchSolver(prob, Cd)
    r = bs.solve(algorithm=alg, iteration_limit=200_000)
    bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
    bs.close()
    return r
for _ in range(10):
    step()
st = torch.cuda.current_stream()
ts = []
for _ in range(300):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); r = step(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(f"{os.environ.get('MPAX_LIB', 'default')}: median {np.median(ts):.4f} ms  min {np.min(ts):.4f}  "
      f"LPs/s {1024 / np.median(ts) * 1e3:.0f}  max it {r['iterations'].max()}  sum att {r['attempts'].sum()}")
