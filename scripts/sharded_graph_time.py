"""Sharded engine per-attempt time with and without the CUDA-graph replay of attempt chunks
(virtual shards on one GPU; C4 = G-RAND(1e5, 2e5, 20, seed 4) by default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("SG_M", "100000"))
lp = lpgen.g_rand(m, 2 * m, 20, seed=4)
for axis in ("rows", "cols"):
    for shards in (1, 2):
        for g in ("1", "0"):
            os.environ["MPAX_SHARDED_GRAPH"] = g
            with mp.ShardedSolver(mp.Problem.from_lp(lp), virtual_shards=shards, axis=axis) as s:
                s.solve(algorithm="ra", iteration_limit=128, eps_abs=0.0, eps_rel=0.0)
                r = s.solve(algorithm="ra", iteration_limit=512, eps_abs=0.0, eps_rel=0.0)
            print(f"{axis} p={shards} graph={g}: {r['solve_seconds'] * 1e6 / r['attempts']:.1f} us/attempt "
                  f"({r['attempts']} attempts)", flush=True)
