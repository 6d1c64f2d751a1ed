"""C5 SpMV pair: the library's standalone pair (lp_spmv_scaled) beside the cuSPARSE yardstick
(bench.py spmv_pair_leg / cusparse_pair_us), printed as one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import lpgen  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

m = int(os.environ.get("C5_M", "5000000"))
lp = lpgen.g_rand(m, 2 * m, 20, seed=5)
prob = mp.Problem.from_lp(lp).to("cuda:0")
peaks = json.load(open(os.path.join(bench.ROOT, "MEASURED_PEAKS.json")))
hbm = peaks.get("hbm_gbs") or 6546.6
print(json.dumps(bench.spmv_pair_leg(mp, torch, "cuda:0", prob, lp, hbm)))
