"""Summarise an ncu report (details page + top stall lines) into markdown."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Block Size", "Grid Size", "Cluster Size",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Dynamic Shared Memory Per Block"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, title):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    seen = {}
    kname = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        kname = d.get("Kernel Name", kname)
        if d.get("Metric Name") in KEYS and d["Metric Name"] not in seen:
            seen[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    rh, ru, rv = raw[0], raw[1], raw[2]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_shared_ld.sum",
            "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_op_dmma.sum", "lts__t_bytes.sum",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]
    rawv = {}
    for i, name in enumerate(rh):
        for w in want:
            if name == w:
                rawv[w] = f"{rv[i]} {ru[i]}"
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    sh = src[1]
    stall_cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    for r in src[2:]:
        for c in stall_cols:
            try:
                tot[c] += int(r[sh.index(c)])
            except (ValueError, IndexError):
                pass
    out = [f"## {title}", "", f"Kernel: `{kname}`", "", "| metric | value |", "|---|---|"]
    out += [f"| {k} | {v} |" for k, v in seen.items()]
    out += [f"| {k} | {v} |" for k, v in rawv.items()]
    s = sum(tot.values()) or 1
    out += ["", "Top warp-stall reasons (share of samples): " +
            ", ".join(f"{k.replace('stall_', '')} {100 * v / s:.0f}%" for k, v in tot.most_common(6)), ""]
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
