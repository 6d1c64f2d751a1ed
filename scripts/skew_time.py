"""Grid-path attempt time on a skewed LP (G-POWERLAW, Pareto row lengths) against G-RAND of the
same shape and about the same nnz: what the row-length skew costs the SpMV mappings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("SK_M", "100000"))
ONLY = os.environ.get("SK_ONLY")
for name, lp in (("uniform", lpgen.g_rand(m, 2 * m, 20, seed=4)),
                 ("powerlaw", lpgen.g_powerlaw(m, 2 * m, 20, seed=9))):
    if ONLY and name != ONLY:
        continue
    lens = np.diff(lp.row_ptr)
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        s.solve(algorithm="ra", path=mp.PATH_GRID, iteration_limit=64, eps_abs=0.0, eps_rel=0.0)
        r = s.solve(algorithm="ra", path=mp.PATH_GRID, iteration_limit=256, eps_abs=0.0, eps_rel=0.0)
    print(f"{name}: nnz {lp.nnz} max row {lens.max()} p99 {np.percentile(lens, 99):.0f}  "
          f"{r['solve_seconds'] * 1e6 / r['attempts']:.1f} us/attempt", flush=True)
