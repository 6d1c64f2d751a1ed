"""lp_create_batch of the C2 batch alone (device inputs): CUDA-event time per call and the
library's host trace (MPAX_HOST_TRACE=1), for A/B of the setup path."""
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
st = torch.cuda.current_stream()
ts = []
for it in range(220):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    bs = mp.BatchSolver(prob, Cd)
    b.record(st)
    torch.cuda.synchronize()
    bs.close()
    if it >= 20:
        ts.append(a.elapsed_time(b) * 1e3)
print(f"{os.path.basename(os.environ.get('MPAX_LIB', 'default'))}: create median {np.median(ts):.1f} us  min {np.min(ts):.1f}")
