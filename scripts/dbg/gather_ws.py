"""Does the gather working set decide the SpMV time?  K~ x with m = 5e6 rows x 20 nnz and
x of n = 2.5e6 .. 1e7 doubles (20 .. 80 MB)."""
import sys; sys.path.insert(0, '.')
import numpy as np, lpgen, torch
import paper_2412_09734_b200 as mp
dev = torch.device("cuda", 0)
for n in (2_500_000, 5_000_000, 7_500_000, 10_000_000):
    lp = lpgen.g_rand(5_000_000, n, 20, seed=5)
    with mp.Solver(mp.Problem.from_lp(lp).to(dev)) as s:
        v = torch.rand(lp.n, dtype=torch.float64, device=dev)
        out = (torch.empty(lp.m, dtype=torch.float64, device=dev), None)
        for _ in range(3):
            s.spmv_scaled(v, None, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            s.spmv_scaled(v, None, out=out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
    print(f"n={n:9d} x={n*8/2**20:5.0f} MB  K~x {ms*1e3:7.1f} us  nnz {lp.nnz}  {lp.nnz/ms/1e6:.2f} Gnnz/s", flush=True)
