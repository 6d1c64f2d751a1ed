"""The bench's SPO+ leg alone (Warcraft-shaped batches), for A/B runs (MPAX_INST_NW etc.)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_09734_b200 as mp  # noqa: E402

ks = tuple(int(k) for k in os.environ.get("SPO_KS", "12,30").split(","))
out = bench.spo_leg(mp, torch, torch.device("cuda", 0), ks=ks)
print(json.dumps({k: {a: v[a]["ms_per_step"] for a in v if isinstance(v[a], dict)} for k, v in out.items()
                  if isinstance(v, dict)}))
