"""profiles/traffic.json from the ncu --set full captures of the benchmarked commit: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch of the C2 register kernel and the C3
DMMA kernel, per attempt of the grid kernel (C4, C5: the capture's solve is limited to PROF_K
accepted steps; the per-attempt figure divides the whole launch -- init, the check at the limit and
the output included -- by its attempts, an upper bound).
usage: python scripts/traffic_from_ncu.py TAG tiny.ncu-rep grid_c4.ncu-rep:ATT grid_c5.ncu-rep:ATT dmma.ncu-rep
       [grid_c5_fp32.ncu-rep:ATT]"""
import csv
import io
import json
import os
import subprocess
import sys


def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        tot += float(v[i]) * scale[u[i]]
    return tot


def main():
    tag, tiny, c4, c5, dm = sys.argv[1:6]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    c4r, c4a = c4.split(":")
    c5r, c5a = c5.split(":")
    out = {"_doc": "DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant kernels from one "
                   f"`ncu --set full --clock-control none` capture each ({tag}, scripts/gpu_round2.sh); bench.py "
                   "copies these into roofline.traffic. Measured under ncu (cold caches, serialised), not live; "
                   "grid figures divide a whole PROF_K-step launch by its attempts (an upper bound).",
           "tiny_kernel_c2": {"bytes_per_launch": dram(tiny), "launch": "one C2 batch solve (1024 LPs, raPDHG, 1e-4)",
                              "capture": os.path.basename(tiny)},
           "grid_kernel_c4": {"bytes_per_attempt": dram(c4r) / float(c4a), "attempts": int(c4a),
                              "algorithmic_bytes_per_attempt": 70.0e6, "capture": os.path.basename(c4r)},
           "grid_kernel_c5": {"bytes_per_attempt": dram(c5r) / float(c5a), "attempts": int(c5a),
                              "algorithmic_bytes_per_attempt": 3.50e9, "capture": os.path.basename(c5r)},
           "dmma_kernel_c3": {"bytes_per_launch": dram(dm), "launch": "one C3 DMMA batch solve",
                              "capture": os.path.basename(dm)}}
    if len(sys.argv) > 6:
        fr, fa = sys.argv[6].split(":")
        out["grid_kernel_c5_fp32"] = {"bytes_per_attempt": dram(fr) / float(fa), "attempts": int(fa),
                                      "algorithmic_bytes_per_attempt": 2.18e9, "capture": os.path.basename(fr)}
    json.dump(out, open(os.path.join(root, "profiles", "traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
