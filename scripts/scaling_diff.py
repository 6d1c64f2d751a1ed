"""GPU vs oracle scalings (Dr, Dc) on the parity LPs: the indices and sizes of any differences."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import lpgen  # noqa: E402
import oracle  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

for name, lp in (("C1", lpgen.g_rand(50, 100, 10, seed=1)), ("ragged", lpgen.g_rand(37, 61, 5, seed=7)),
                 ("dense", lpgen.g_dense(30, 50, batch=1, seed=5)[0]), ("grid", lpgen.g_grid(batch=1)[0])):
    with mp.Solver(mp.Problem.from_lp(lp)) as s:
        Dr, Dc = s.scaling()
    Dro, Dco = oracle.precondition(lp)
    for lab, a, b in (("Dr", Dr, Dro), ("Dc", Dc, Dco)):
        d = np.nonzero(a != b)[0]
        rel = np.max(np.abs(a - b) / np.abs(b)) if d.size else 0.0
        print(f"{os.environ.get('MPAX_SETUP_STOP', '0')} {name:7s} {lab}: {d.size} of {a.size} differ, max rel {rel:.2e}, first {d[:6]}")
