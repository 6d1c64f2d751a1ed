"""C1 (G-RAND(50, 100, 10, seed 1), r2HPDHG to 1e-4): the whole path per LP and the solve kernel time,
for A/B of the single-LP kernels (MPAX_LIB, MPAX_INST_NW)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

lp = lpgen.g_rand(50, 100, 10, seed=1)
prob = mp.Problem.from_lp(lp).to("cuda:0")
st = torch.cuda.current_stream()
ts, ks = [], []
alg = os.environ.get("C1_ALG", "r2")
for rep in range(int(os.environ.get("C1_REPS", 105))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with mp.Solver(prob) as s:
        r = s.solve(algorithm=alg)
        s.solution(memory=mp.LP_DEVICE)
    e1.record(st)
    torch.cuda.synchronize()
    if rep >= 5:
        ts.append(e0.elapsed_time(e1) * 1e3)
        ks.append(r["solve_seconds"] * 1e6)
print(f"{os.path.basename(os.environ.get('MPAX_LIB', 'default'))} NW={os.environ.get('MPAX_INST_NW', '-')} {alg}: "
      f"path {np.median(ts):.1f} us  solve {np.median(ks):.1f} us  it {r['iterations']} att {r['attempts']} "
      f"us/att {np.median(ks) / r['attempts']:.2f} status {r['status']}", flush=True)
