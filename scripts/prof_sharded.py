"""C5 (or SG_M-sized) LP on the sharded engine at one NCCL rank, a short fixed-K solve: run under
`ncu --metrics gpu__time_duration.sum` for the per-kernel split of a sharded attempt."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("SG_M", "5000000"))
axis = os.environ.get("SG_AXIS", "rows")
k = int(os.environ.get("SG_K", "32"))
lp = lpgen.g_rand(m, 2 * m, 20, seed=5 if m == 5_000_000 else 4)
full = mp.Problem.from_lp(lp)
loc = (mp.local_cols(full, 0, lp.n) if axis == "cols" else full).to("cuda")
comm = mp.nccl_comm_init(1, mp.nccl_unique_id(), 0)
kw = dict(axis="cols", n_global=lp.n) if axis == "cols" else dict(m1_global=lp.m1, m2_global=lp.m2)
with mp.ShardedSolver(loc, comm=comm, rank=0, nranks=1, **kw) as s:
    for _ in range(2):
        r = s.solve(algorithm="ra", iteration_limit=k, eps_abs=0.0, eps_rel=0.0)
    print(f"{axis}: {r['solve_seconds'] * 1e6 / r['attempts']:.1f} us/attempt ({r['attempts']} attempts)", flush=True)
mp.nccl_comm_destroy(comm)
