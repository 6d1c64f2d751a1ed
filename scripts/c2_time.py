"""C2 step timing only (bench.py's step: create + batch solve + solutions + close), for A/B runs
of the library (MPAX_LIB).  Prints the median step, the median solve (the library's own event
time around the solver launch) and the slowest instance's attempts (the critical path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

lp, C = bench.make_workload(int(os.environ.get("C2_BATCH", 1024)), seed=2)
B = C.shape[0]
dev = torch.device("cuda", 0)
prob = mp.Problem.from_lp(lp).to(dev)
Cd = torch.as_tensor(C, device=dev)
X = torch.empty((B, lp.n), dtype=torch.float64, device=dev)
Y = torch.empty((B, lp.m), dtype=torch.float64, device=dev)
alg = os.environ.get("C2_ALG", "ra")
rule = os.environ.get("C2_RULE", "adaptive")


def step():
    bs = mp.BatchSolver(prob, Cd)
    r = bs.solve(algorithm=alg, iteration_limit=200_000, step_rule=rule)
    bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
    bs.close()
    return r


for _ in range(10):
    step()
st = torch.cuda.current_stream()
# C2_FLUSH=1: evict L2 between steps (outside the event pair), as bench.py's timed region does
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev) if os.environ.get("C2_FLUSH") else None
ts, ss = [], []
# C2_NOSYNC=1: no host synchronisation between steps (bench.py's timed loop); C2_NOGC=1: Python's
# cyclic garbage collector off during the loop
if os.environ.get("C2_NOGC"):
    import gc
    gc.collect()
    gc.disable()
nosync = bool(os.environ.get("C2_NOSYNC"))
evs = []
for _ in range(int(os.environ.get("C2_REPS", 300))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if flush is not None:
        flush.zero_()
    a.record(st); r = step(); b.record(st)
    if not nosync:
        torch.cuda.synchronize()
    evs.append((a, b)); ss.append(float(r["solve_seconds"][0]) * 1e3)
torch.cuda.synchronize()
ts = [a.elapsed_time(b) for a, b in evs]
print(f"mean step {np.mean(ts):.4f} ms  p90 {np.percentile(ts, 90):.4f}  max {np.max(ts):.4f}", flush=True)
att = int(r["attempts"].max())
print(f"{os.path.basename(os.environ.get('MPAX_LIB', 'default')):12s} {'cold' if flush is not None else 'warm'} {alg} step {np.median(ts):.4f} ms (min {np.min(ts):.4f})  "
      f"solve {np.median(ss):.4f} ms  LPs/s {B / np.median(ts) * 1e3:.0f}  max it {r['iterations'].max()}  "
      f"max att {att} (instance {int(np.argmax(r['attempts']))})  us/att {np.median(ss) * 1e3 / att:.3f}  sum att {r['attempts'].sum()}", flush=True)
