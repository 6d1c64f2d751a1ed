"""Replace the C5 grid-kernel entries of profiles/traffic.json by the MARGINAL DRAM traffic per
attempt: two launches limited to K = 16 and 32 accepted steps (scripts/gpu_c5_marginal.sh; same
init, check and output), so (T32 - T16) / 16 counts the attempts alone.
usage: python scripts/traffic_marginal.py gpurun_out/c5m"""
import csv
import io
import json
import os
import sys


def dram(f):
    lines = [ln for ln in open(f).read().splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    return tot


def main(prefix):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", "traffic.json")
    out = json.load(open(path))
    for key, prec, alg_bytes in (("grid_kernel_c5", "fp64", 3.50e9), ("grid_kernel_c5_fp32", "fp32", 2.18e9)):
        a, b = dram(f"{prefix}_{prec}_16.csv"), dram(f"{prefix}_{prec}_32.csv")
        out[key] = {"bytes_per_attempt": (b - a) / 16, "algorithmic_bytes_per_attempt": alg_bytes,
                    "method": "marginal: (DRAM bytes of a 32-step launch - a 16-step launch) / 16, "
                              "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (scripts/gpu_c5_marginal.sh)",
                    "launch_16_bytes": a, "launch_32_bytes": b}
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("grid_kernel_c5", "grid_kernel_c5_fp32")}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
